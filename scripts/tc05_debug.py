"""Time the tcgen05 fused conv on cfg2 with roles switched off
(NENT_TC05_DEBUG bits: 1 producer math, 2 epilogue math, 4 MMAs)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

rng = np.random.default_rng(5)
n, K = 1 << 24, 256
x = torch.from_numpy(rng.integers(-2048, 2048, (3, n), dtype=np.int64)).cuda().to(torch.int32)
g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
p = nent.derive_params(3, int(os.environ.get("NENT_W", "64")))
fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
gd = D.taps_tensor(g, fl)
L = n + K - 1
if os.environ.get("NENT_PAD"):  # 128-byte aligned output rows (padded pitch)
    out = torch.empty((3, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
else:
    out = torch.empty((3, L), dtype=torch.int32, device="cuda")
for dbg in [int(a) for a in sys.argv[1:]] or range(8):
    os.environ["NENT_TC05_DEBUG"] = str(dbg)
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, None, True, n + K - 1, n_in=n, out=out)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print("debug", dbg, "ms", round(e0.elapsed_time(e1) / 10, 4), flush=True)
