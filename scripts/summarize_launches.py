"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import re
import sys


def summarize(path):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ix = {h: k for k, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        short = re.sub(r"\(.*", "", r[ix["Kernel Name"]])[:80]
        ns = float(r[ix["Metric Value"]].replace(",", ""))
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    out = [f"{len(rows) - 1} launches, {tot / 1e6:.3f} ms total (cold-cache, serialised under ncu)",
           "", "| launches | total ms | share | kernel |", "|---:|---:|---:|---|"]
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {c} | {ns / 1e6:.3f} | {100 * ns / tot:.1f}% | `{k}` |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
