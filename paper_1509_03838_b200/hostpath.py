"""Host-buffer path of the fused hot path: pinned host in, pinned host out.

This is what a caller holding plain host arrays goes through (the e2e number
of bench.py).  The signal is cut into output chunks; each chunk's input slice
(+ K-1 halo) is copied host->device, convolved by the fused
entangle->conv->extract kernel, and copied back.  Three streams form a
three-stage pipeline -- H2D copies, kernels, D2H copies -- over a ring of
device buffers, ordered by CUDA events, so both copy engines and the SMs stay
busy concurrently: the job time approaches max(H2D bytes, D2H bytes) / PCIe
bandwidth plus one chunk of fill and drain.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from .errors import ParameterError
from .params import CodecParams


class ChunkedEntangledConv:
    """Reusable pipeline for one geometry: m streams of n samples, K taps.

    Inputs/outputs are pinned host tensors (int32 or int64); outputs are the
    recovered full-convolution samples, n + K - 1 per stream."""

    def __init__(self, params: CodecParams, n: int, g, flavor: int, chunk: int = 1 << 21,
                 in_dtype=torch.int32, out_dtype=torch.int32, nbuf: int = 4,
                 device: torch.device | None = None):
        self.p = params
        self.n = n
        self.g = np.asarray(g, dtype=np.int64)
        self.K = len(self.g)
        self.L = n + self.K - 1
        self.flavor = flavor
        self.chunk = min(chunk, self.L)
        self.in_dtype, self.out_dtype = in_dtype, out_dtype
        self.dev = device or D.device()
        self.g_dev = D.taps_tensor(self.g, flavor)
        m, H = params.m, self.K - 1
        self.table = D.imma_table(self.g_dev, self.K, flavor, y_begin=H)  # every chunk starts at H
        self.s_in = torch.cuda.Stream(device=self.dev)
        self.s_comp = torch.cuda.Stream(device=self.dev)
        self.s_out = torch.cuda.Stream(device=self.dev)
        self.nbuf = nbuf
        self.xbuf = [torch.empty((m, self.chunk + H), dtype=in_dtype, device=self.dev) for _ in range(nbuf)]
        self.ybuf = [torch.empty((m, self.chunk), dtype=out_dtype, device=self.dev) for _ in range(nbuf)]
        self.launches = 0

    def chunks(self):
        for s in range(0, self.L, self.chunk):
            yield s, min(s + self.chunk, self.L)

    def h2d_bytes(self) -> int:
        es = torch.tensor([], dtype=self.in_dtype).element_size()
        return self.p.m * self.n * es  # every input sample crosses once (halo re-reads aside)

    def d2h_bytes(self) -> int:
        es = torch.tensor([], dtype=self.out_dtype).element_size()
        return self.p.m * self.L * es

    def run(self, c_host: torch.Tensor, d_host: torch.Tensor, failed: int | None = None) -> int:
        """Enqueue the whole job; returns the number of kernels launched.
        Call ``synchronize()`` before reading ``d_host``."""
        if not c_host.is_pinned() or not d_host.is_pinned():
            raise ParameterError("host buffers must be pinned (torch.empty(..., pin_memory=True))")
        m, H, n = self.p.m, self.K - 1, self.n
        in_done = [torch.cuda.Event() for _ in range(self.nbuf)]
        comp_done = [None] * self.nbuf
        out_done = [None] * self.nbuf
        launches = 0
        for idx, (s, e) in enumerate(self.chunks()):
            k = idx % self.nbuf
            xb, yb = self.xbuf[k], self.ybuf[k]
            lo, hi = s - H, e  # input window [lo, hi) of this chunk
            a, b = max(lo, 0), min(hi, n)
            width = hi - lo
            with torch.cuda.stream(self.s_in):
                if comp_done[k] is not None:  # the kernel that last read xb has finished
                    self.s_in.wait_event(comp_done[k])
                if lo < 0 or hi > n:
                    xb[:, :width].zero_()
                if b > a:
                    for i in range(m):
                        xb[i, a - lo:b - lo].copy_(c_host[i, a:b], non_blocking=True)
                in_done[k].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(in_done[k])
                if out_done[k] is not None:  # the copy that last read yb has finished
                    self.s_comp.wait_event(out_done[k])
                D.fused_conv(xb[:, :width], self.g_dev, self.K, self.p.l, self.flavor, failed,
                             self.p.w > 32, period=width, n_in=width, y_begin=H, n_out=e - s,
                             out=yb[:, : e - s], imma_table=self.table)
                launches += 1
                comp_done[k] = torch.cuda.Event()
                comp_done[k].record(self.s_comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(comp_done[k])
                for i in range(m):
                    d_host[i, s:e].copy_(yb[i, : e - s], non_blocking=True)
                out_done[k] = torch.cuda.Event()
                out_done[k].record(self.s_out)
        self.launches = launches
        return launches

    def synchronize(self):
        for st in (self.s_in, self.s_comp, self.s_out):
            st.synchronize()

    def capture(self, c_host: torch.Tensor, d_host: torch.Tensor, failed: int | None = None):
        """Record the whole job (every copy, kernel and cross-stream event) as
        one CUDA graph on these host buffers; ``replay()`` then costs a single
        launch instead of ~8 host calls per chunk."""
        self.run(c_host, d_host, failed)  # warm: allocator, kernel attributes, tables
        self.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=self.dev)
        with torch.cuda.graph(self.graph, stream=cap):
            for st in (self.s_in, self.s_comp, self.s_out):  # fork into the capture
                st.wait_stream(cap)
            self.run(c_host, d_host, failed)
            for st in (self.s_in, self.s_comp, self.s_out):  # join back
                cap.wait_stream(st)
        torch.cuda.synchronize(self.dev)
        return self.graph

    def replay(self):
        self.graph.replay()
