"""cfg5 two-pass chain: time interleave, gather_chain and the fused conv separately."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _device as D, fused, workloads  # noqa: E402
from paper_1509_03838_b200._lib import MAC_NAMES, call, ptr, row_ptrs  # noqa: E402

dev = torch.device("cuda", 0)
wl = workloads.make(5)
p = wl.params
c = torch.from_numpy(wl.c).to(dev).to(torch.int32)
n, K, m = wl.n, wl.K, wl.m
L = n + K - 1
a = torch.from_numpy(wl.add).to(dev)
add = D.shift_add(a, a, p.l)
perm = torch.from_numpy(wl.perm).to(dev)
perm32 = perm.to(torch.int32)
xb = int(np.abs(wl.c).max()) * ((1 << p.l) + 1) * abs(wl.scale) + int(add.abs().max())
ct = torch.empty((n, m), dtype=torch.int32, device=dev)
xg = torch.empty((m, n), dtype=torch.int32, device=dev)
out = torch.empty((m, L), dtype=torch.int32, device=dev)
fl = fused.conv_flavor(xb, wl.g, n_out=L)
gd = D.taps_tensor(wl.g, fl)
tab = D.imma_table(gd, K, fl, 0)
print("params", p, "flavor", MAC_NAMES[fl], "kernel", D.imma_kernel(fl, K, m, True), "x bound", xb)
steps = {
    "interleave": lambda: call("nent_interleave", row_ptrs(c), 32, m, n, ptr(ct), D._sh()),
    "gather_chain": lambda: D.gather_chain(ct, p.l, wl.scale, add, perm, out=xg),
    "interleave_chain": lambda: D.interleave_chain(c, p.l, wl.scale, add, out=ct),
    "gather_records32": lambda: D.gather_records(ct, perm32, out=xg),
    "fused_conv": lambda: D.fused_conv(xg, gd, K, p.l, fl, None, True, L, n_in=n, out=out, pre_entangled=True,
                                       imma_table=tab),
}
for name, f in steps.items():
    f()
torch.cuda.synchronize()
for name, f in steps.items():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(name, "ms", e0.elapsed_time(e1) / 5)

# alternative conv stage: tcgen05 plain conv of the 8 chain rows, then K3 extract
fl_tc = fl  # same digits (imma2x1); plain mode runs on tcgen05 for <= 64 rows
print("plain kernel for 8 rows:", D.imma_kernel(fl_tc, K, m, False))
delta = torch.empty((m, L), dtype=torch.int32, device=dev)
dout = torch.empty((m, L), dtype=torch.int32, device=dev)
alt = {
    "tc05_plain_conv": lambda: D.conv(xg, gd, K, fl_tc, period=L, n_out=L, out=delta),
    "extract_K3": lambda: D.extract(delta, m, p.l, 0, False, out=dout),
}
for name, f in alt.items():
    f()
torch.cuda.synchronize()
for name, f in alt.items():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(name, "ms", e0.elapsed_time(e1) / 5)
steps["fused_conv"]()
torch.cuda.synchronize()
print("same result:", torch.equal(dout, out))
