"""The cfg2 m = 3 kernel launched right behind a 1 ms CUDA-core (F64) plain convolution, each m3
launch timed on its own (the position of `entangled` in bench.py's interleaved loop).  With a
stamps build (`--dump`) the last launch's per-CTA timeline is printed."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200 import fused, workloads  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 11
dump = "--dump" in sys.argv
wl = workloads.make(2)
n, K = wl.n, wl.K
L = n + K - 1
p = nent.derive_params(3, 48)
x = torch.from_numpy(wl.c).cuda().to(torch.int32)
fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
core = fused.conv_flavor(2048 * ((1 << p.l) + 1), wl.g, allow_imma=False)
gd, gc = D.taps_tensor(wl.g, fl), D.taps_tensor(wl.g, core)
out = torch.empty((3, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
yp = torch.empty((3, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
f = lambda: D.fused_conv(x, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm)  # noqa: E731
pred = sys.argv[sys.argv.index("--pred") + 1] if "--pred" in sys.argv else "f64"
plain_fl = imma_flavor(2, 2)
gp = D.taps_tensor(wl.g, plain_fl)
h = {"f64": lambda: D.conv(x, gc, K, core, period=L, n_out=L, out=yp),
     "failed": lambda: D.fused_conv(x, gd, K, p.l, fl, 1, True, L, n_in=n, out=out),
     "plainfast": lambda: D.conv(x, gp, K, plain_fl, period=L, n_out=L, out=yp),
     "generic": lambda: D.conv(x, gd, K, fl, period=L, n_out=L, out=yp)}[pred]
f(); h()
torch.cuda.synchronize()
evs = []
for i in range(reps):
    h()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if dump and i == reps - 1:
        os.environ["NENT_M3_DUMP"] = "1"
    f()
    e1.record()
    evs.append((e0, e1))
torch.cuda.synchronize()
ts = [a.elapsed_time(b) for a, b in evs]
print("m3 behind", pred, D.last_conv_kernel(), ": median", round(statistics.median(ts), 4), "min", round(min(ts), 4), "max", round(max(ts), 4), flush=True)
