"""Quick GPU probe: fused cfg2 conv with each exact flavour, timed with CUDA
events, checked against the known-answer digest."""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D, fused, workloads  # noqa: E402
from paper_1509_03838_b200._lib import MAC_F64, MAC_I32, MAC_NAMES, MAC_S64, imma_flavor  # noqa: E402

digests = json.loads((Path(__file__).resolve().parents[1] / "tests/golden/digests.json").read_text())


def sha(t):
    return hashlib.sha256(np.ascontiguousarray(t.to(torch.int64).cpu().numpy(), dtype="<i8").tobytes()).hexdigest()


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


CFGS = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]
for cfg in CFGS:
    wl = workloads.make(cfg)
    p = wl.params
    c = torch.from_numpy(wl.c).cuda().to(torch.int32)
    n, K = wl.n, wl.K
    L = n + K - 1
    out = torch.empty((wl.m, L), dtype=torch.int32, device="cuda")
    mc = int(np.abs(wl.c).max())
    xb = mc * ((1 << p.l) + 1)
    add = perm = None
    scale = 1
    if wl.scale is not None:
        scale = wl.scale
        a_dev = torch.from_numpy(wl.add).cuda()
        add = D.shift_add(a_dev, a_dev, p.l)
        perm = torch.from_numpy(wl.perm).cuda()
        xb = xb * abs(scale) + int(add.abs().max())
    np_, ng = D.signed_digits(xb), D.signed_digits(int(np.abs(wl.g).max()))
    cands = [imma_flavor(np_, ng), D.cuda_core_flavor(xb, int(np.abs(wl.g).sum()), int(np.abs(wl.g).max()))]
    res = {}
    for fl in cands:
        gd = D.taps_tensor(wl.g, fl)
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")

        def run():
            D.fused_conv(c, gd, K, p.l, fl, None, p.w > 32, L, n_in=n, out=out, mismatch=mm,
                         scale=scale, add=add, perm=perm)
        t = bench(run)
        ok = sha(out) == digests[f"cfg{cfg}"]["d"]
        mm.zero_()
        run()
        torch.cuda.synchronize()
        res[MAC_NAMES[fl]] = {"ms": round(t, 4), "exact": ok, "mismatch": int(mm.item()),
                             "samples_per_s": wl.m * L / (t / 1e3), "gmac_s": wl.m * n * K / (t / 1e3) / 1e9}
    # plain narrowest
    gpl = D.pick_flavor(mc if wl.scale is None else mc * abs(scale) + 128, int(np.abs(wl.g).sum()),
                        int(np.abs(wl.g).max()), K=K)
    print(json.dumps({"cfg": cfg, "np": np_, "ng": ng, "results": res, "plain_pick": MAC_NAMES[gpl]}))
