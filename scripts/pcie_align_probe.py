"""Does host-side address alignment change pinned DMA throughput?  4 MiB
row copies (the e2e pipeline's size) at host offsets 0 / 1 / 16 / 255 words,
H2D alone, D2H alone, and both directions concurrently."""
import json
import time

import torch

W = 1 << 20  # words per copy
NC = 48      # copies per direction (201 MB, like cfg2)
h_in = torch.empty(NC * W + 8192, dtype=torch.int32).pin_memory()
h_out = torch.empty(NC * W + 8192, dtype=torch.int32).pin_memory()
d_in = torch.empty(NC * W + 8192, dtype=torch.int32, device="cuda")
d_out = torch.empty(NC * W + 8192, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


res = {}
import sys
sizes = [W]
offs = [(0, 0), (1, 0), (16, 0), (64, 0), (256, 0), (1024, 0), (4096, 0), (1024, 3)]
for hoff, doff in offs:
    def h2d():
        with torch.cuda.stream(s1):
            for k in range(NC):
                d_in[doff + k * W:doff + (k + 1) * W].copy_(h_in[hoff + k * W:hoff + (k + 1) * W], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            for k in range(NC):
                h_out[hoff + k * W:hoff + (k + 1) * W].copy_(d_out[doff + k * W:doff + (k + 1) * W], non_blocking=True)

    def both():
        h2d()
        d2h()
    res[f"host+{hoff}_dev+{doff}"] = {"h2d_ms": timed(h2d), "d2h_ms": timed(d2h), "both_ms": timed(both)}
# aligned starts, ragged sizes
for sz in (W - 1, W - 255, W + 17):
    def both_sz():
        with torch.cuda.stream(s1):
            for k in range(NC):
                d_in[k * W:k * W + sz].copy_(h_in[k * W:k * W + sz], non_blocking=True)
        with torch.cuda.stream(s2):
            for k in range(NC):
                h_out[k * W:k * W + sz].copy_(d_out[k * W:k * W + sz], non_blocking=True)
    res[f"aligned_size{sz}"] = {"both_ms": timed(both_sz)}
print(json.dumps(res, indent=1))
