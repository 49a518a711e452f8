"""PCIe probe of the e2e pipeline's access pattern: 3 host rows of 2^24 int32
each way, copied in chunks either row by row (1-D copies, rows interleaved
per chunk) or as one 2-D copy per chunk (cudaMemcpy2DAsync), H2D and D2H
concurrently on two streams; plus the one-big-copy floor."""
import json
import time

import torch
from cuda.bindings import runtime as rt

M, N = 3, 1 << 24
h_in = torch.zeros((M, N), dtype=torch.int32).pin_memory()
h_out = torch.zeros((M, N), dtype=torch.int32).pin_memory()
d_in = torch.zeros((M, N), dtype=torch.int32, device="cuda")
d_out = torch.zeros((M, N), dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


res = {}


def whole():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


res["whole_both"] = timed(whole)
for chunk in (1 << 19, 1 << 20, 1 << 21, 1 << 22):
    def rows1d():
        for s in range(0, N, chunk):
            with torch.cuda.stream(s1):
                for i in range(M):
                    d_in[i, s:s + chunk].copy_(h_in[i, s:s + chunk], non_blocking=True)
            with torch.cuda.stream(s2):
                for i in range(M):
                    h_out[i, s:s + chunk].copy_(d_out[i, s:s + chunk], non_blocking=True)

    def rows2d():
        for s in range(0, N, chunk):
            rt.cudaMemcpy2DAsync(d_in.data_ptr() + 4 * s, N * 4, h_in.data_ptr() + 4 * s, N * 4, chunk * 4, M,
                                 H2D, s1.cuda_stream)
            rt.cudaMemcpy2DAsync(h_out.data_ptr() + 4 * s, N * 4, d_out.data_ptr() + 4 * s, N * 4, chunk * 4, M,
                                 D2H, s2.cuda_stream)

    def rows_sep_streams():  # each row its own pair of streams
        for s in range(0, N, chunk):
            for i in range(M):
                with torch.cuda.stream(ss_in[i]):
                    d_in[i, s:s + chunk].copy_(h_in[i, s:s + chunk], non_blocking=True)
                with torch.cuda.stream(ss_out[i]):
                    h_out[i, s:s + chunk].copy_(d_out[i, s:s + chunk], non_blocking=True)
    ss_in = [torch.cuda.Stream() for _ in range(M)]
    ss_out = [torch.cuda.Stream() for _ in range(M)]
    res[f"chunk{chunk}"] = {"rows1d": timed(rows1d), "rows2d": timed(rows2d),
                            "rows_sep_streams": timed(rows_sep_streams)}
print(json.dumps(res, indent=1))
