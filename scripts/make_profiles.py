"""Turn one evidence run (gpurun_out/<TAG>_*, written by scripts/gpu_round.sh)
into the tracked files under profiles/: bench lines, launch-list summary, the
ncu raw page of the headline kernel, its per-role source summary and the
DRAM traffic entry bench.py reads.  Usage: python scripts/make_profiles.py TAG"""
import csv
import json
import re
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO / "scripts"))
from summarize_launches import summarize  # noqa: E402

tag = sys.argv[1]
G, P = REPO / "gpurun_out", REPO / "profiles"


def last_json(path):
    lines = [ln for ln in path.read_text().splitlines() if ln.startswith("{")]
    return lines[-1] if lines else None


for src, dst in ((f"{tag}_bench.log", f"{tag}_bench_cfg2.jsonl"), (f"{tag}_ref.log", f"{tag}_bench_reference_arm.jsonl")):
    ln = last_json(G / src) if (G / src).exists() else None
    if ln:
        (P / dst).write_text(ln + "\n")
if (G / f"{tag}_launches.csv").exists():
    (P / f"{tag}_launches.csv").write_text((G / f"{tag}_launches.csv").read_text())
    (P / f"{tag}_launches.md").write_text(summarize(G / f"{tag}_launches.csv") + "\n")
rep = G / f"{tag}_prof_m3.ncu-rep"
if rep.exists():
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    (P / f"{tag}_ncu_raw_tcgen05_m3_cfg2.csv").write_text(raw)
    rows = list(csv.reader(raw.splitlines()))
    hdr, val = rows[0], rows[2]
    get = lambda k: float(val[hdr.index(k)].replace(",", ""))  # noqa: E731
    unit = lambda k: rows[1][hdr.index(k)]  # noqa: E731
    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}
    rd = get("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
    wr = get("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
    tf = P / "ncu_traffic.json"
    t = json.loads(tf.read_text()) if tf.exists() else {}
    t["tcgen05_m3"] = {"bytes_per_launch": int(rd + wr),
                       "note": f"dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture of "
                               f"tcm3::conv_tc05_m3_kernel<2,12> on cfg2 (profiles/{tag}_ncu_raw_tcgen05_m3_cfg2.csv): "
                               f"{rd / 1e6:.2f} MB read + {wr / 1e6:.2f} MB written (the rest of the 201 MB output "
                               "still dirty in L2 at kernel end)"}
    tf.write_text(json.dumps(t, indent=1) + "\n")
    src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    tmp = Path("/tmp") / f"{tag}_src.csv"
    tmp.write_text(src)
    out = subprocess.run([sys.executable, str(REPO / "scripts" / "ncu_src_summary.py"), str(tmp), "30"],
                         capture_output=True, text=True).stdout
    out = re.sub(r"0x[0-9a-f]{8,}", lambda m: "0x.." + m.group(0)[-5:], out)
    (P / f"{tag}_ncu_source_roles.txt").write_text(
        "regions: 0 = setup (before setmaxnreg), 1 = epilogue warps, 2 = converters + loader + MMA issuer\n" + out)
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.max", "sm__cycles_active.avg", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "gpc__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
            "sm__inst_executed.avg.per_cycle_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    print({k: (val[hdr.index(k)], unit(k)) for k in keys if k in hdr})

rep4 = G / f"{tag}_prof_m4.ncu-rep"
if rep4.exists():
    raw = subprocess.run(["ncu", "-i", str(rep4), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    (P / f"{tag}_ncu_raw_tcgen05_m4_cfg3.csv").write_text(raw)
    rows = list(csv.reader(raw.splitlines()))
    hdr, val = rows[0], rows[2]
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.max", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.avg.per_second"]
    print("m4:", {k: (val[hdr.index(k)], rows[1][hdr.index(k)]) for k in keys if k in hdr})
