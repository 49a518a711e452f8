"""One cfg2-sized fused conv launch per kernel flavour (for ncu captures)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

mma_sync = "--mma-sync" in sys.argv
rng = np.random.default_rng(5)
n, K = 1 << 24, 256
x = torch.from_numpy(rng.integers(-2048, 2048, (3, n), dtype=np.int64)).cuda().to(torch.int32)
g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
p = nent.derive_params(3, 48 if "--w48" in sys.argv else 64)
fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048), mma_sync)
gd = D.taps_tensor(g, fl)
out = torch.empty((3, n + K - 1), dtype=torch.int32, device="cuda")
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    D.fused_conv(x, gd, K, p.l, fl, None, True, n + K - 1, n_in=n, out=out, mismatch=mm)
torch.cuda.synchronize()
print("mismatch", int(mm.item()))
