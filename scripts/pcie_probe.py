"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (2 streams),
to size the e2e path of bench.py."""
import json
import time

import torch

n = 3 * (1 << 24)  # cfg2: 3 streams of 2^24 int32 = 201 MB
h_in = torch.empty(n, dtype=torch.int32).pin_memory()
h_out = torch.empty(n, dtype=torch.int32).pin_memory()
d_in = torch.empty(n, dtype=torch.int32, device="cuda")
d_out = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both_concurrent", both)):
    t = timed(fn)
    res[name] = {"ms": t * 1e3, "GB_s_each_direction": n * 4 / t / 1e9}
for chunks in (4, 8, 16, 32):
    step = n // chunks

    def chunked():
        for k in range(chunks):
            st = s1 if k % 2 == 0 else s2
            with torch.cuda.stream(st):
                d_in[k * step:(k + 1) * step].copy_(h_in[k * step:(k + 1) * step], non_blocking=True)
                h_out[k * step:(k + 1) * step].copy_(d_out[k * step:(k + 1) * step], non_blocking=True)
    t = timed(chunked)
    res[f"chunked_{chunks}"] = {"ms": t * 1e3}
print(json.dumps(res))
