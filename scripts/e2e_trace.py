"""CUPTI timeline (torch.profiler) of one eager ChunkedEntangledConv job on
the cfg2 geometry: per-stream memcpy / kernel intervals, written as a compact
JSON for offline analysis of the pipeline's bubbles."""
import json
import sys
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import fused  # noqa: E402
from paper_1509_03838_b200.hostpath import ChunkedEntangledConv  # noqa: E402
from bench import make_inputs  # noqa: E402

chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
n, K = 1 << 24, 256
params, c_np, g = make_inputs(0, n, K)
m, H = params.m, K - 1
flavor = fused.conv_flavor(int(np.abs(c_np).max()) * ((1 << params.l) + 1), g, n_out=n + H)
c_host = torch.from_numpy(c_np.astype(np.int32)).pin_memory()
d_host = torch.empty((m, n + H), dtype=torch.int32).pin_memory()
pipe = ChunkedEntangledConv(params, n, g, flavor, chunk=chunk)
for _ in range(2):
    pipe.run(c_host, d_host)
    pipe.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pipe.run(c_host, d_host)
    pipe.synchronize()
Path("gpurun_out").mkdir(exist_ok=True)
prof.export_chrome_trace(f"gpurun_out/e2e_trace_{chunk}.json")
ev = json.load(open(f"gpurun_out/e2e_trace_{chunk}.json"))["traceEvents"]
rows = []
for e in ev:
    if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"):
        rows.append({"cat": e["cat"], "name": e["name"][:40], "ts": e["ts"], "dur": e.get("dur", 0),
                     "stream": e.get("args", {}).get("stream")})
rows.sort(key=lambda r: r["ts"])
t0 = rows[0]["ts"]
for r in rows:
    r["ts"] = round(r["ts"] - t0, 1)
json.dump(rows, open(f"gpurun_out/e2e_rows_{chunk}.json", "w"))
span = max(r["ts"] + r["dur"] for r in rows)
by = {}
for r in rows:
    k = (r["cat"], r["stream"])
    by.setdefault(k, [0, 0.0])
    by[k][0] += 1
    by[k][1] += r["dur"]
print("span_us", span)
for k, v in sorted(by.items(), key=str):
    print(k, "n", v[0], "busy_us", round(v[1], 1))
