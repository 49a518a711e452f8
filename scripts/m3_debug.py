"""Small fused m = 3 (l = 16) launches for debugging the conv_tc05_m3 kernel."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rng = np.random.default_rng(1)
c = rng.integers(-2048, 2048, (3, n), dtype=np.int64)
g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
p = nent.derive_params(3, 48)
x = torch.from_numpy(c).cuda().to(torch.int32)
fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
gd = D.taps_tensor(g, fl)
L = n + K - 1
out = torch.empty((3, L), dtype=torch.int32, device="cuda")
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
D.fused_conv(x, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm)
print("kernel", D.last_conv_kernel(), flush=True)
torch.cuda.synchronize()
ref = O.full_conv(c, g)
got = out.to(torch.int64).cpu().numpy()
bad = np.argwhere(got != ref)
print("mismatch", int(mm.item()), "bad", len(bad), bad[:5].tolist())
