"""Repeat every tcgen05 kernel of the round many times on fixed inputs and
check that each launch reproduces the first launch's (oracle-checked
elsewhere) output bit for bit and that the redundant-stream check stays at
zero: a synchronisation race would show up as a differing launch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(123)


def repeat(name, launch, out, mm):
    launch()
    torch.cuda.synchronize()
    first = out.clone()
    bad = 0
    for i in range(reps):
        out.fill_(-1)
        launch()
        if not torch.equal(out, first):
            bad += 1
    torch.cuda.synchronize()
    print(f"{name}: {reps} launches, {bad} differing, mismatch counter {int(mm.item()) if mm is not None else 0},"
          f" kernel {D.last_conv_kernel()}", flush=True)
    return bad == 0 and (mm is None or int(mm.item()) == 0)


ok = True
# m = 3 fused (verify, failed) and plain, several sizes incl. ragged ones
for n, K in ((1 << 22, 256), (3 * 8192 + 77, 129), (1 << 20, 64)):
    p = nent.derive_params(3, 48)
    c = torch.from_numpy(rng.integers(-2048, 2048, (3, n))).cuda().to(torch.int32)
    g = rng.integers(-2048, 2048, (K,))
    fl = imma_flavor(4, 2)
    gd = D.taps_tensor(g, fl)
    L = n + K - 1
    out = torch.empty((3, L), dtype=torch.int32, device="cuda")
    for r in (None, 1):
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")
        ok &= repeat(f"m3 fused n={n} K={K} r={r}",
                     lambda: D.fused_conv(c, gd, K, p.l, fl, r, True, L, n_in=n, out=out,
                                          mismatch=mm if r is None else None), out, mm)
    flp = imma_flavor(2, 2)
    gp = D.taps_tensor(g, flp)
    ok &= repeat(f"m3 plain n={n} K={K}", lambda: D.conv(c, gp, K, flp, period=L, n_out=L, out=out), out, None)
# m = 4 long filter
for n, K in ((1 << 21, 1024), (5 * 4096 + 77, 300)):
    p = nent.derive_params(4, 64)
    c = torch.from_numpy(rng.integers(-512, 512, (4, n))).cuda().to(torch.int32)
    g = rng.integers(-512, 512, (K,))
    fl = imma_flavor(4, 2)
    gd = D.taps_tensor(g, fl)
    L = n + K - 1
    out = torch.empty((4, L), dtype=torch.int32, device="cuda")
    for r in (None, 2):
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")
        ok &= repeat(f"m4 fused n={n} K={K} r={r}",
                     lambda: D.fused_conv(c, gd, K, p.l, fl, r, True, L, n_in=n, out=out,
                                          mismatch=mm if r is None else None), out, mm)
# m = 8 pre-entangled
for n, K in ((1 << 21, 128), (3 * 4096 + 77, 257)):
    p = nent.derive_params(8, 32)
    cc = rng.integers(-100, 100, (8, n))
    eps = (np.roll(cc, 1, axis=0) << p.l) + cc
    x = torch.from_numpy(eps).cuda().to(torch.int32)
    g = rng.integers(-100, 100, (K,))
    fl = imma_flavor(2, 1)
    gd = D.taps_tensor(g, fl)
    L = n + K - 1
    out = torch.empty((8, L), dtype=torch.int32, device="cuda")
    for r in (None, 5):
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")
        ok &= repeat(f"m8 fused n={n} K={K} r={r}",
                     lambda: D.fused_conv(x, gd, K, p.l, fl, r, False, L, n_in=n, out=out,
                                          mismatch=mm if r is None else None, pre_entangled=True), out, mm)
print("STRESS", "OK" if ok else "FAILED")
sys.exit(0 if ok else 1)
