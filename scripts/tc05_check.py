"""tcgen05 conv kernel vs the mma.sync kernel vs the CPU oracle: plain and
fused (m = 3, every failure + verify), small and cfg2-sized, plus timing."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D, fused  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor, MAC_NAMES  # noqa: E402
from oracle import oracle as O  # noqa: E402

O.build()
rng = np.random.default_rng(5)
ok = True
for n, K in [(3000, 77), (100000, 256), (9000, 1), (20000, 64), (5000, 200)]:
    x = rng.integers(-2048, 2048, (3, n), dtype=np.int64)
    g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
    ref = O.full_conv(x, g)
    for mma_sync in (False, True):
        fl = imma_flavor(D.signed_digits(2048), D.signed_digits(2048), mma_sync)
        y, _ = D.conv(torch.from_numpy(x).cuda().to(torch.int32), D.taps_tensor(g, fl), K, fl, period=n + K - 1)
        same = np.array_equal(y.cpu().numpy(), ref)
        ok &= same
        print("plain", n, K, MAC_NAMES[fl], same, flush=True)
    p = nent.derive_params(3, 64)
    eb = 2048 * ((1 << p.l) + 1)
    for mma_sync in (False, True):
        fl = imma_flavor(D.signed_digits(eb), D.signed_digits(2048), mma_sync)
        for r in (None, 0, 1, 2):
            res = fused.entangled_conv(nent.StreamBlock(p, torch.from_numpy(x).cuda().to(torch.int32)), g,
                                       failed=r, flavor=fl)
            same = np.array_equal(res.outputs.data.cpu().numpy(), ref)
            ok &= same and (r is not None or res.mismatches == 0)
            print("fused", n, K, MAC_NAMES[fl], r, same, res.mismatches, flush=True)

# cfg2 timing
n, K = 1 << 24, 256
x = torch.from_numpy(rng.integers(-2048, 2048, (3, n), dtype=np.int64)).cuda().to(torch.int32)
g = rng.integers(-2048, 2048, (K,), dtype=np.int64)
p = nent.derive_params(3, 64)
eb = 2048 * ((1 << p.l) + 1)
outs = {}
for mma_sync in (False, True):
    fl = imma_flavor(D.signed_digits(eb), D.signed_digits(2048), mma_sync)
    gd = D.taps_tensor(g, fl)
    out = torch.empty((3, n + K - 1), dtype=torch.int32, device="cuda")
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, None, True, n + K - 1, n_in=n, out=out, mismatch=mm)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    outs[mma_sync] = out.clone()
    print("cfg2 fused", MAC_NAMES[fl], "ms", e0.elapsed_time(e1) / 10, "mismatch", int(mm.item()), flush=True)
same = torch.equal(outs[False], outs[True])
ok &= same
print("cfg2 tc05 == mma.sync:", same)
print("ALL OK" if ok else "FAIL")
