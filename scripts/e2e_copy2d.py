"""e2e pipeline with one 2-D DMA per chunk and direction (cudaMemcpy2DAsync
through cuda-python) instead of one copy per row: does it close the gap to
the pure-copy floor?  Diagnostic only."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import fused, hostpath  # noqa: E402
from bench import make_inputs, sha  # noqa: E402

H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


class Pipe2D(hostpath.ChunkedEntangledConv):
    def _h2d(self, xb, c_host, lo, a, b):
        es = c_host.element_size()
        a0 = max(a - self._lead(c_host, 0, a), 0)
        rt.cudaMemcpy2DAsync(xb.data_ptr() + (hostpath.PRE + a0 - lo) * es, xb.stride(0) * es,
                             c_host.data_ptr() + a0 * es, c_host.stride(0) * es, (b - a0) * es, self.p.m,
                             H2D, torch.cuda.current_stream().cuda_stream)

    def _d2h(self, d_host, yb, h0s, h1s, ys):
        es = d_host.element_size()
        h0, h1 = h0s[0], h1s[0]
        if h1 > h0:
            rt.cudaMemcpy2DAsync(d_host.data_ptr() + h0 * es, d_host.stride(0) * es,
                                 yb.data_ptr() + (h0 - ys) * es, yb.stride(0) * es, (h1 - h0) * es, self.p.m,
                                 D2H, torch.cuda.current_stream().cuda_stream)


n, K = 1 << 24, 256
params, c_np, g = make_inputs(0, n, K)
m, H = params.m, K - 1
dev = torch.device("cuda", 0)
flavor = fused.conv_flavor(int(np.abs(c_np).max()) * ((1 << params.l) + 1), g, n_out=n + H)
c_host = torch.from_numpy(c_np.astype(np.int32)).pin_memory()
res = {}


def wall(fn, reps=8):
    fn()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
        torch.cuda.synchronize(dev)
    return (time.perf_counter() - t0) / reps * 1e3


ref = None
for pad in (0, 1):  # pad=1: d_host rows 256-byte aligned (row stride rounded up)
    Lp = n + H if not pad else (n + H + 63) // 64 * 64
    d_full = torch.empty((m, Lp), dtype=torch.int32).pin_memory()
    d_host = d_full[:, :n + H]
    for cls in (hostpath.ChunkedEntangledConv, Pipe2D):
        for chunk in (1 << 18, 1 << 19, 1 << 20, 1 << 21):
            for lag in (1, 2):
                pipe = cls(params, n, g, flavor, chunk=chunk, lag=lag, ramp=0)
                pipe.capture(c_host, d_host)
                t = wall(pipe.replay)
                h = sha(d_host.to(torch.int64).numpy())
                ref = ref or h
                res[f"{cls.__name__}_pad{pad}_chunk{chunk}_lag{lag}"] = [round(t, 3), h == ref]
                del pipe
print(json.dumps(res, indent=1))
