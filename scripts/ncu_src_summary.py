"""Summarise an ncu --page source --csv --print-source sass export: per-role
(region between USETMAXREG markers) executed instructions and stall samples,
and the hottest instructions."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try:
        return float(r[ix[k]].replace(",", "") or 0)
    except (ValueError, IndexError):
        return 0.0
region = 0
agg = collections.defaultdict(lambda: collections.Counter())
hot = []
for r in data:
    src = r[ix["Source"]]
    if "USETMAXREG" in src:
        region += 1
    a = agg[region]
    a["inst"] += num(r, "Instructions Executed")
    a["samples"] += num(r, "Warp Stall Sampling (All Samples)")
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            a[k] += num(r, k)
    op = src.split()[0] if src.split() else ""
    if op.startswith("@"):
        op = src.split()[1]
    a["op:" + op] += num(r, "Instructions Executed")
    hot.append((num(r, "Warp Stall Sampling (All Samples)"), num(r, "Instructions Executed"), r[ix["Address"]], src[:70],
                {k: num(r, k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k and num(r, k) > 0}))
for reg, a in sorted(agg.items()):
    print(f"region {reg}: inst {a['inst']:.3g} samples {a['samples']:.3g}")
    st = sorted(((v, k) for k, v in a.items() if k.startswith("stall_")), reverse=True)[:8]
    print("   stalls:", ", ".join(f"{k[6:]}={v:.0f}" for v, k in st))
    ops = sorted(((v, k) for k, v in a.items() if k.startswith("op:")), reverse=True)[:14]
    print("   ops:", ", ".join(f"{k[3:]}={v:.3g}" for v, k in ops))
hot.sort(reverse=True)
for s, n, ad, src, st in hot[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s:7.0f} {n:9.0f} {ad} {src:70s} {top}")
