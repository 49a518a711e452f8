"""The cfg3 m = 4 kernel (and cfg5's m = 8 conv stage with --m8) launched right behind another
kernel that leaves the L2 full of its own dirty output (a plain conv into another buffer), each
launch timed on its own: the position kernels have in bench.py's interleaved loop."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200 import workloads  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

reps = 21
if "--m8" in sys.argv:
    n, K = 1 << 24, 128
    p = nent.derive_params(8, 32)
    rng = np.random.default_rng(5)
    g = rng.integers(-3, 4, (K,), dtype=np.int64)
    c = torch.from_numpy(rng.integers(-8, 8, (8, n), dtype=np.int32)).cuda()
    x = c + (torch.roll(c, 1, 0) << p.l)
    fl = imma_flavor(2, 1)
    gd = D.taps_tensor(g, fl)
    L = n + K - 1
    out = torch.empty((8, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, None, False, L, n_in=n, out=out, mismatch=mm, pre_entangled=True)  # noqa: E731
else:
    wl = workloads.make(3)
    n, K, p = wl.n, wl.K, wl.params
    L = n + K - 1
    x = torch.from_numpy(wl.c).cuda().to(torch.int32)
    fl = imma_flavor(4, 2)
    gd = D.taps_tensor(wl.g, fl)
    out = torch.empty((4, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm)  # noqa: E731
# predecessor: a plain 3 x 2^24 K = 256 conv into its own buffer (201 MB of output)
w2 = workloads.make(2)
x2 = torch.from_numpy(w2.c).cuda().to(torch.int32)
pf = imma_flavor(2, 2)
g2 = D.taps_tensor(w2.g, pf)
L2 = w2.n + w2.K - 1
y2 = torch.empty((3, (L2 + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L2]
h = lambda: D.conv(x2, g2, w2.K, pf, period=L2, n_out=L2, out=y2)  # noqa: E731
f(); h()
torch.cuda.synchronize()
evs = []
for i in range(reps):
    h()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f()
    e1.record()
    evs.append((e0, e1))
torch.cuda.synchronize()
ts = [a.elapsed_time(b) for a, b in evs]
print(D.last_conv_kernel(), "behind a plain conv: median", round(statistics.median(ts), 4), "min", round(min(ts), 4), flush=True)
