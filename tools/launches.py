"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel).
Usage: python tools/launches.py launches.csv [skip_first_n_launches]"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    if int(r[ii]) < skip or r[mi] != "gpu__time_duration.sum":
        continue
    per[(int(r[ii]), r[ki].split("(")[0][:50])] = float(r[vi].replace(",", "")) / 1000.0
agg = collections.defaultdict(lambda: [0, 0.0])
for (i, k), us in per.items():
    agg[k][0] += 1
    agg[k][1] += us
tot = sum(v[1] for v in agg.values())
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {n:5d} {us / n:10.1f} us  {us / tot:6.3f}")
