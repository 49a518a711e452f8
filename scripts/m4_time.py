"""Time the cfg3 fused m = 4 long-filter kernel (verify and failed = 1) at full size."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200 import workloads  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

import os  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dump = "--dump" in sys.argv  # stamps builds (-DNENT_M4_STAMPS): the timeline of one more back-to-back launch
wl = workloads.make(3)
n, K, p = wl.n, wl.K, wl.params
L = n + K - 1
x = torch.from_numpy(wl.c).cuda().to(torch.int32)
fl = imma_flavor(4, 2)
gd = D.taps_tensor(wl.g, fl)
out = torch.empty((4, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
for r in (None, 1):
    f = lambda: D.fused_conv(x, gd, K, p.l, fl, r, True, L, n_in=n, out=out, mismatch=mm if r is None else None)  # noqa
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    if dump:
        os.environ["NENT_M4_DUMP"] = "1"
        f()
        del os.environ["NENT_M4_DUMP"]
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    macs = 4 * n * K * 8 * (1 if r is None else 0.75)
    print("failed", r, "kernel", D.last_conv_kernel(), "ms", round(ms, 4), "digit TMAC/s", round(macs / ms / 1e9, 1),
          "mismatch", int(mm.item()), flush=True)
