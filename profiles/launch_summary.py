"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, mean duration and share of the library's kernel time per kernel.
Usage: python profiles/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
kn, mn, mv, un = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if r[mn] != "gpu__time_duration.sum":
        continue
    v = float(r[mv].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[un]]
    name = r[kn].split("(")[0].removeprefix("void ")
    agg[name].append(v * scale)
dfc_total = sum(sum(v) for k, v in agg.items() if k.startswith("dfc::"))
print(f"{'kernel':45s} {'launches':>8s} {'mean us':>9s} {'share of dfc time':>18s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = sum(v) / dfc_total if k.startswith("dfc::") else float("nan")
    print(f"{k[:45]:45s} {len(v):8d} {sum(v) / len(v):9.1f} {share:18.3f}")
