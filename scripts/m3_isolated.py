"""Isolated-launch time of the cfg2 m = 3 kernel: every launch timed on its own with CUDA events,
a 512 MB fill in between (cold L2), median of N.  `python scripts/m3_isolated.py [N]`."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200 import workloads  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
wl = workloads.make(2)
n, K = wl.n, wl.K
L = n + K - 1
p = nent.derive_params(3, 48)
x = torch.from_numpy(wl.c).cuda().to(torch.int32)
fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
gd = D.taps_tensor(wl.g, fl)
out = torch.empty((3, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
junk = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for r in (None, 1):
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, r, True, L, n_in=n, out=out, mismatch=mm if r is None else None)  # noqa
    f()
    ts = []
    for _ in range(reps):
        junk.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("failed", r, "isolated ms: median", round(statistics.median(ts), 4), "min", round(min(ts), 4), flush=True)
