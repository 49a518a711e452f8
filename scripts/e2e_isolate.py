"""Isolate the e2e pipeline's overhead: the same ChunkedEntangledConv job
(graph replay) with the fused kernel, with no kernel at all (copies + event
dependencies only), and with a sleep kernel of the same duration."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _device as D, fused, hostpath  # noqa: E402
from bench import make_inputs  # noqa: E402

n, K = 1 << 24, 256
params, c_np, g = make_inputs(0, n, K)
m, H = params.m, K - 1
dev = torch.device("cuda", 0)
flavor = fused.conv_flavor(int(np.abs(c_np).max()) * ((1 << params.l) + 1), g, n_out=n + H)
c_host = torch.from_numpy(c_np.astype(np.int32)).pin_memory()
d_host = torch.empty((m, n + H), dtype=torch.int32).pin_memory()
real = D.fused_conv
res = {}


def wall(fn, reps=8):
    fn()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
        torch.cuda.synchronize(dev)
    return (time.perf_counter() - t0) / reps * 1e3


for chunk, lag, ramp, variant in [(c, lg, rp, v) for c in (1 << 20, 1 << 21, 1 << 22) for lg in (0, 1, 2)
                                  for rp in (0, 4) for v in ("real", "nokernel")]:
    if True:
        if variant == "nokernel":
            hostpath.D.fused_conv = lambda *a, **k: None
        elif variant == "sleep":
            cyc = int(1.9e9 * 42e-6 * chunk / (1 << 20))  # ~42 us per 2^20 outputs
            hostpath.D.fused_conv = lambda *a, **k: torch.cuda._sleep(cyc)
        else:
            hostpath.D.fused_conv = real
        pipe = hostpath.ChunkedEntangledConv(params, n, g, flavor, chunk=chunk, lag=lag, ramp=ramp)
        pipe.capture(c_host, d_host)
        res[f"chunk{chunk}_lag{lag}_ramp{ramp}_{variant}"] = wall(pipe.replay)
        del pipe
hostpath.D.fused_conv = real
print(json.dumps(res, indent=1))
