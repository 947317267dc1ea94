"""Summarise the kernels of an ncu --set full report as JSON (the fields DESIGN.md
and bench.py's traffic entries cite).  Usage:
    python profiles/ncu_to_json.py report.ncu-rep "command that produced it" > out.json"""
import csv
import json
import subprocess
import sys

rep, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
FIELDS = ["SM Frequency", "Memory Throughput", "DRAM Throughput", "Duration", "Executed Ipc Active",
          "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
          "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
          "Achieved Occupancy", "L2 Cache Throughput", "L1/TEX Cache Throughput"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"]


def rows(page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


res = {}
d = rows("details")
h = d[0]
ids, kn, sec, mn, mu, mv = (h.index(x) for x in ("ID", "Kernel Name", "Section Name", "Metric Name",
                                                 "Metric Unit", "Metric Value"))
gi, bi = h.index("Grid Size"), h.index("Block Size")
for r in d[1:]:
    k = f"launch {r[ids]}"
    e = res.setdefault(k, {"command": cmd, "kernel": r[kn], "block": r[bi], "grid": r[gi]})
    if r[mn] in FIELDS and r[mn] not in e:
        e[r[mn]] = f"{r[mv]} {r[mu]}".strip()
raw = rows("raw")
hdr, units = raw[0], raw[1]
for n, r in enumerate(raw[2:]):
    e = res.get(f"launch {r[hdr.index('ID')]}")
    if e is None:
        continue
    for m in RAW:
        if m in hdr:
            e[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
json.dump(res, sys.stdout, indent=1)
print()
