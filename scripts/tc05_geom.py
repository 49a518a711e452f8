"""A/B of the cfg2 codec geometry on the tcgen05 fused kernel:
(3,64,21,21) -> 5 digit planes vs (3,48,16,16) -> 4 planes.
Times the fused entangled launch and the same kernel on the plain streams
(back to back, CUDA events), and checks the recovered outputs' digest."""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200 import workloads  # noqa: E402
from paper_1509_03838_b200._lib import MAC_NAMES, imma_flavor  # noqa: E402

REPO = Path(__file__).resolve().parents[1]
known = json.loads((REPO / "tests" / "golden" / "digests.json").read_text())["cfg2"]["d"]
wl = workloads.make(2)
n, K = wl.n, wl.K
L = n + K - 1
x = torch.from_numpy(wl.c).cuda().to(torch.int32)
pitch = (L + 31) // 32 * 32
out = torch.empty((3, pitch), dtype=torch.int32, device="cuda")[:, :L]
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50


def timeit(f):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for w in (64, 48):
    p = nent.derive_params(3, w)
    fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
    gd = D.taps_tensor(wl.g, fl)
    tab = D.imma_table(gd, K, fl, 0)
    fused = lambda: D.fused_conv(x, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm,  # noqa: E731
                                 imma_table=tab)
    failed = lambda: D.fused_conv(x, gd, K, p.l, fl, 1, True, L, n_in=n, out=out, imma_table=tab)  # noqa: E731
    plain = lambda: D.conv(x, gd, K, fl, period=L, n_out=L, out=out, imma_table=tab)  # noqa: E731
    mm.zero_()
    fused()
    torch.cuda.synchronize()
    dig = hashlib.sha256(np.ascontiguousarray(out.to(torch.int64).cpu().numpy(), dtype="<i8").tobytes()).hexdigest()
    ok = dig == known and int(mm.item()) == 0
    res = {}
    for rnd in range(3):
        for name, f in (("fused", fused), ("plain_same", plain), ("failed_r1", failed)):
            res.setdefault(name, []).append(timeit(f))
    med = {k: float(np.median(v)) for k, v in res.items()}
    print(json.dumps({"w": w, "l": p.l, "flavor": MAC_NAMES[fl], "kernel": D.imma_kernel(fl, K, 3, True),
                      "exact": ok, "ms": med,
                      "overhead_pct": (med["fused"] - med["plain_same"]) / med["plain_same"] * 100}), flush=True)
