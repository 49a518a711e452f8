"""Clocks, power and throttle reasons (NVML) while the cfg2 m = 3 kernel runs back to back
for a few seconds: `python scripts/power_probe.py [seconds]`."""
import sys
import time
from pathlib import Path

import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1509_03838_b200 as nent  # noqa: E402
from paper_1509_03838_b200 import _device as D  # noqa: E402
from paper_1509_03838_b200 import workloads  # noqa: E402
from paper_1509_03838_b200._lib import imma_flavor  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
wl = workloads.make(2)
n, K = wl.n, wl.K
L = n + K - 1
p = nent.derive_params(3, 48)
x = torch.from_numpy(wl.c).cuda().to(torch.int32)
fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
gd = D.taps_tensor(wl.g, fl)
out = torch.empty((3, (L + 31) // 32 * 32), dtype=torch.int32, device="cuda")[:, :L]
mm = torch.zeros(1, dtype=torch.int64, device="cuda")
f = lambda: D.fused_conv(x, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm)  # noqa: E731
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
print("power limit W", pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3, flush=True)
f()
torch.cuda.synchronize()
t_end = time.time() + secs
launches = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
while time.time() < t_end:
    e0.record()
    for _ in range(400):
        f()
    e1.record()
    launches += 400
    time.sleep(0.02)  # the queue is ~40 ms deep: sample mid-way
    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1e3
    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    tp = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
    torch.cuda.synchronize()
    print(f"sm {sm} MHz power {pw:.0f} W temp {tp} C reasons {rs:#x} ms/launch {e0.elapsed_time(e1) / 400:.4f}", flush=True)
