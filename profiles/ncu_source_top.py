"""Summarise an ncu report's source page: top CUDA lines by executed
instructions and by warp-stall samples.  Usage: python ncu_source_top.py rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, out, hdr = None, [], None
for r in csv.reader(txt.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].isdigit():
        num = lambda k: int(r[hdr.index(k)]) if r[hdr.index(k)].isdigit() else 0
        ie = num("Instructions Executed")
        sm = num("Warp Stall Sampling (All Samples)")
        if ie or sm:
            out.append((ie, sm, cur, int(r[0]), r[1][:95]))
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"total warp-instructions {tot}  stall samples {ts}")
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0]:>11} {100*o[0]/tot:5.1f}%  stall {100*o[1]/ts:5.1f}%  {o[2]}:{o[3]}  {o[4]}")
