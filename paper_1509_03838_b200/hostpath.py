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


PRE = 64    # device lead-in words before each input window (host reads start 256-byte aligned)
LEAD = 64   # extra outputs computed before each chunk (host writes start 256-byte aligned)
ALIGN = 256  # pinned DMA runs at full duplex rate only from/to 256-byte-aligned host addresses


class ChunkedEntangledConv:
    """Reusable pipeline for one geometry: m streams of n samples, K taps.

    Inputs/outputs are pinned host tensors (int32 or int64); outputs are the
    recovered full-convolution samples, n + K - 1 per stream.

    Each chunk moves as ONE 2-D DMA per direction (all m rows, nent_copy_rows)
    -- per-row copies cost ~5% at 2^20-sample chunks and ~20% at 2^18.  Host
    transfers start on a 256-byte boundary (row 0's; other rows follow the
    caller's pitch): concurrent H2D + D2H loses ~20% when the host side is
    misaligned (profiles/r01_e2e_pipeline.md), so each input copy starts at the
    aligned word at or below its window (the kernel reads its rows from
    ``PRE`` words in), and each chunk computes ``LEAD`` extra outputs before
    its window so its output copy can start at the aligned word at or below
    the chunk boundary.  ``ramp`` > 0 shrinks the first and last chunks
    (chunk / 2^ramp ...); with the output lag below it does not pay on cfg2.

    Output copies lag the input copies by ``lag`` chunks (chunk j's D2H also
    waits for chunk j + lag's H2D).  Without it the two directions run in
    lockstep -- H2D(j+1) and D2H(j) share the link and finish together -- and
    every chunk's kernel then sits exposed on the D2H stream: an idle output
    direction does not make the input direction much faster, so the input
    side never builds the lead that would hide it (profiles/r01_e2e_pipeline.md)."""

    def __init__(self, params: CodecParams, n: int, g, flavor: int, chunk: int = 1 << 20,
                 in_dtype=torch.int32, out_dtype=torch.int32, nbuf: int = 4,
                 device: torch.device | None = None, ramp: int = 0, lag: int = 1):
        self.p = params
        self.n = n
        self.g = np.asarray(g, dtype=np.int64)
        self.K = len(self.g)
        self.L = n + self.K - 1
        self.flavor = flavor
        self.bounds = self._schedule(self.L, max(chunk, 1024), ramp)
        self.chunk = max(e - s for s, e in self.bounds)
        self.in_dtype, self.out_dtype = in_dtype, out_dtype
        self.dev = device or D.device()
        self.g_dev = D.taps_tensor(self.g, flavor)
        m, H = params.m, self.K - 1
        # every chunk's input window starts HP = K-1 rounded up to 4 samples before
        # its first output, so the kernel's tiles start on 16-byte boundaries
        self.HP = (H + 3) // 4 * 4
        self.table = D.imma_table(self.g_dev, self.K, flavor, y_begin=self.HP)
        self.s_in = torch.cuda.Stream(device=self.dev)
        self.s_comp = torch.cuda.Stream(device=self.dev)
        self.s_out = torch.cuda.Stream(device=self.dev)
        if not 0 <= lag < nbuf:
            raise ParameterError(f"lag {lag} must be in [0, nbuf)")
        self.nbuf, self.lag = nbuf, lag
        row = (PRE + LEAD + self.chunk + self.HP + 31) // 32 * 32  # 128-byte row starts
        self.xbuf = [torch.empty((m, row), dtype=in_dtype, device=self.dev) for _ in range(nbuf)]
        self.ybuf = [torch.empty((m, LEAD + self.chunk), dtype=out_dtype, device=self.dev)
                     for _ in range(nbuf)]
        self.launches = 0

    @staticmethod
    def _schedule(L: int, chunk: int, ramp: int) -> list[tuple[int, int]]:
        head = [chunk >> k for k in range(ramp, 0, -1) if chunk >> k >= 4096]
        if 2 * sum(head) + chunk > L:
            head = []
        mid = L - 2 * sum(head)
        nmid = max(1, -(-mid // chunk))
        step = ((mid + nmid - 1) // nmid + 63) // 64 * 64 if nmid > 1 else mid
        sizes = head + [step] * (nmid - 1) + [mid - step * (nmid - 1)] + head[::-1]
        out, s = [], 0
        for z in sizes:
            if z > 0:
                out.append((s, s + z))
                s += z
        assert s == L
        return out

    def chunks(self):
        yield from self.bounds

    def h2d_bytes(self) -> int:
        es = torch.tensor([], dtype=self.in_dtype).element_size()
        return self.p.m * self.n * es  # every input sample crosses once (halo re-reads aside)

    def d2h_bytes(self) -> int:
        es = torch.tensor([], dtype=self.out_dtype).element_size()
        return self.p.m * self.L * es

    @staticmethod
    def _lead(t: torch.Tensor, i: int, j: int) -> int:
        """Words between t[i, j] and the 256-byte boundary at or below it."""
        addr = t.data_ptr() + (i * t.stride(0) + j * t.stride(1)) * t.element_size()
        return (addr % ALIGN) // t.element_size()

    def _h2d(self, xb, c_host, lo, a, b):
        """Input window [a, b) of every row -> xb (device word PRE + p - lo
        holds sample p), one 2-D DMA starting at row 0's aligned word."""
        a0 = max(a - self._lead(c_host, 0, a), 0)
        D.copy_rows(xb[:, PRE + a0 - lo:PRE + b - lo], c_host[:, a0:b])

    def _d2h(self, d_host, yb, h0, h1, ys):
        """Outputs [h0, h1) of every row -> host (yb word q holds ys + q)."""
        if h1 > h0:
            D.copy_rows(d_host[:, h0:h1], yb[:, h0 - ys:h1 - ys])

    def _check_host(self, c_host: torch.Tensor, d_host: torch.Tensor):
        m, n, L = self.p.m, self.n, self.L
        if not c_host.is_pinned() or not d_host.is_pinned():
            raise ParameterError("host buffers must be pinned (torch.empty(..., pin_memory=True))")
        if tuple(c_host.shape) != (m, n) or tuple(d_host.shape) != (m, L):
            raise ParameterError(f"expected c_host {(m, n)} and d_host {(m, L)}")
        if c_host.stride(1) != 1 or d_host.stride(1) != 1:
            raise ParameterError("host rows must be contiguous")

    def run(self, c_host: torch.Tensor, d_host: torch.Tensor, failed: int | None = None) -> int:
        """Enqueue the whole job; returns the number of kernels launched.
        Call ``synchronize()`` before reading ``d_host``."""
        return self.run_many([(c_host, d_host)], failed)

    def run_many(self, jobs, failed: int | None = None) -> int:
        """Enqueue several jobs ((c_host, d_host) pairs) as one continuous
        chunk pipeline: the next job's first input copies overlap the previous
        job's last kernels and output copies, so the pipeline fills and drains
        once for the whole batch of jobs instead of once per job."""
        for c_host, d_host in jobs:
            self._check_host(c_host, d_host)
        n, H = self.n, self.HP
        seq = [(jb, s, e) for jb in range(len(jobs)) for (s, e) in self.bounds]
        nch = len(seq)
        in_ev = [torch.cuda.Event() for _ in range(nch)]
        comp_ev = [torch.cuda.Event() for _ in range(nch)]
        out_ev = [torch.cuda.Event() for _ in range(nch)]
        # output copy starts: row 0's aligned word at or below each chunk boundary
        hs = []
        for _, d_host in jobs:
            hs.append([0] + [max(s - self._lead(d_host, 0, s), 0) for s, _ in self.bounds[1:]] + [self.L])
        nb = len(self.bounds)

        def d2h(j):
            """Copy chunk j's outputs back once its kernel is done and, with
            lag, once the input of chunk j + lag has arrived."""
            jb, s, e = seq[j]
            ci = j - jb * nb  # chunk index within its job
            ys = max(s - LEAD, 0)
            yb = self.ybuf[j % self.nbuf]
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(comp_ev[j])
                if j + self.lag < nch:
                    self.s_out.wait_event(in_ev[j + self.lag])
                self._d2h(jobs[jb][1], yb, hs[jb][ci], hs[jb][ci + 1], ys)
                out_ev[j].record(self.s_out)

        launches = 0
        for idx, (jb, s, e) in enumerate(seq):
            c_host = jobs[jb][0]
            k = idx % self.nbuf
            xb, yb = self.xbuf[k], self.ybuf[k]
            ys = max(s - LEAD, 0)  # this chunk's outputs [ys, e)
            lo, hi = ys - H, e     # and its input window [lo, hi)
            a, b = max(lo, 0), min(hi, n)
            width = hi - lo
            with torch.cuda.stream(self.s_in):
                if idx >= self.nbuf:  # the kernel that last read xb has finished
                    self.s_in.wait_event(comp_ev[idx - self.nbuf])
                if lo < 0:
                    xb[:, PRE:PRE - lo].zero_()
                if hi > n:
                    xb[:, PRE + max(n - lo, 0):PRE + width].zero_()
                if b > a:
                    self._h2d(xb, c_host, lo, a, b)
                in_ev[idx].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(in_ev[idx])
                if idx >= self.nbuf:  # the copy that last read yb has finished
                    self.s_comp.wait_event(out_ev[idx - self.nbuf])
                D.fused_conv(xb[:, PRE:PRE + width], self.g_dev, self.K, self.p.l, self.flavor, failed,
                             self.p.w > 32, period=width, n_in=width, y_begin=H, n_out=e - ys,
                             out=yb[:, : e - ys], imma_table=self.table)
                launches += 1
                comp_ev[idx].record(self.s_comp)
            if idx - self.lag >= 0:
                d2h(idx - self.lag)
        for j in range(max(nch - self.lag, 0), nch):
            d2h(j)
        self.launches = launches
        return launches

    def synchronize(self):
        for st in (self.s_in, self.s_comp, self.s_out):
            st.synchronize()

    def capture(self, c_host: torch.Tensor, d_host: torch.Tensor, failed: int | None = None,
                jobs: int = 1):
        """Record the whole job (every copy, kernel and cross-stream event) as
        one CUDA graph on these host buffers; ``replay()`` then costs a single
        launch instead of ~8 host calls per chunk.  ``jobs`` > 1 records that
        many back-to-back jobs on the same buffers as one continuous pipeline
        (``run_many``): a stream of batches, filled and drained once."""
        self.run(c_host, d_host, failed)  # warm: allocator, kernel attributes, tables
        self.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=self.dev)
        with torch.cuda.graph(self.graph, stream=cap):
            for st in (self.s_in, self.s_comp, self.s_out):  # fork into the capture
                st.wait_stream(cap)
            self.run_many([(c_host, d_host)] * jobs, failed)
            for st in (self.s_in, self.s_comp, self.s_out):  # join back
                cap.wait_stream(st)
        torch.cuda.synchronize(self.dev)
        return self.graph

    def replay(self):
        self.graph.replay()
