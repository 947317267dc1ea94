"""Attribute an ncu source page to code regions of a kernel file by line ranges
(found from marker comments).  Usage: python ncu_phase_split.py rep [k_rows.cu]"""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
srcname = sys.argv[2] if len(sys.argv) > 2 else "k_rows.cu"
src = open("paper_2106_03503_b200/csrc/" + srcname).read().splitlines()
marks = []
for n, line in enumerate(src, 1):
    m = re.search(r"// ---- (\d\. [^-]+|[0-9]\.)", line)
    if "struct RowCtx" in line:
        marks.append((n, "RowCtx (merge lookups/walk)"))
    if "__global__ void __launch_bounds__" in line:
        marks.append((n, "kernel prologue"))
    if m:
        marks.append((n, m.group(1).strip()))
marks.sort()
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
for r in csv.reader(txt.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].isdigit():
        v = lambda k: int(r[hdr.index(k)]) if r[hdr.index(k)].isdigit() else 0
        ln = int(r[0])
        key = "helpers:" + cur
        if cur == srcname:
            key = "header"
            for n, name in marks:
                if ln >= n:
                    key = name
        a = agg.setdefault(key, [0, 0, 0])
        a[0] += v("Instructions Executed")
        a[1] += v("Thread Instructions Executed")
        a[2] += v("Warp Stall Sampling (All Samples)")
tot = sum(a[0] for a in agg.values()) or 1
ts = sum(a[2] for a in agg.values()) or 1
for k, (ie, ti, st) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:34s} {ie/1e6:8.1f}M warp-inst {100*ie/tot:5.1f}%  lanes {ti/max(ie,1):5.1f}  stall-samples {100*st/ts:5.1f}%")
