"""Time cfg5's convolution stage alone: the fused m = 8 kernel on eight already-entangled
int32 rows of 2^24 samples (K = 128), verify and failed = 3."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n, K = 1 << 24, 128
p = nent.derive_params(8, 32)
rng = np.random.default_rng(5)
g = rng.integers(-3, 4, (K,), dtype=np.int64)
c = torch.from_numpy(rng.integers(-8, 8, (8, n), dtype=np.int32)).cuda()
x = c + (torch.roll(c, 1, 0) << p.l)  # rows already entangled
fl = imma_flavor(2, 1)
gd = D.taps_tensor(g, fl)
L = n + K - 1
out = torch.empty((8, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
for r in (None, 3):
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, r, False, L, n_in=n, out=out, mismatch=mm if r is None else None,  # noqa
                             pre_entangled=True)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print("failed", r, "kernel", D.last_conv_kernel(), "ms", round(ms, 4), "GB/s", round(2 * 8 * n * 4 / ms / 1e6, 1),
          "mismatch", int(mm.item()), flush=True)
