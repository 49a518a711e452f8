"""Sweep ChunkedEntangledConv chunk size / ring depth on the cfg2 geometry
(graph replay vs eager), next to the raw pinned copy times, to locate the gap
between the e2e time and the PCIe floor."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _device as D, fused  # noqa: E402
from paper_1509_03838_b200.hostpath import ChunkedEntangledConv  # noqa: E402
from paper_1509_03838_b200._lib import MAC_NAMES  # noqa: E402
from bench import make_inputs  # noqa: E402

n, K = 1 << 24, 256
params, c_np, g = make_inputs(0, n, K)
m, H = params.m, K - 1
dev = torch.device("cuda", 0)
flavor = fused.conv_flavor(int(np.abs(c_np).max()) * ((1 << params.l) + 1), g, n_out=n + H)
c_host = torch.from_numpy(c_np.astype(np.int32)).pin_memory()
d_host = torch.empty((m, n + H), dtype=torch.int32).pin_memory()
res = {"flavor": MAC_NAMES[flavor]}


def wall(fn, reps=8):
    fn()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
        torch.cuda.synchronize(dev)
    return (time.perf_counter() - t0) / reps * 1e3


ref = None
for chunk in (1 << 20, 1 << 21, 1 << 22):
    for ramp in (0, 3, 5):
        nbuf = 4
        pipe = ChunkedEntangledConv(params, n, g, flavor, chunk=chunk, nbuf=nbuf, ramp=ramp)
        eager = wall(lambda: pipe.run(c_host, d_host))
        pipe.capture(c_host, d_host)
        graph = wall(pipe.replay)
        out = d_host.numpy().copy()
        if ref is None:
            ref = out
        res[f"chunk{chunk}_ramp{ramp}"] = {"eager_ms": eager, "graph_ms": graph,
                                           "same": bool(np.array_equal(out, ref))}
        del pipe
        torch.cuda.empty_cache()
# one kernel over the whole resident signal, for the compute share
x = torch.from_numpy(c_np.astype(np.int32)).to(dev)
gd = D.taps_tensor(g, flavor)
y = torch.empty((m, n + H), dtype=torch.int32, device=dev)
tab = D.imma_table(gd, K, flavor, y_begin=0)


def kern():
    D.fused_conv(x, gd, K, params.l, flavor, None, False, n + H, n_in=n, out=y, imma_table=tab)


res["resident_kernel_ms"] = wall(kern)
print(json.dumps(res, indent=1))
