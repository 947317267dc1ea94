"""End-to-end time of the C++ drop-in: host BinaryImage in ->
edt() -> host DistanceMap (uint64) out, per call, through lib/dropin_cli
time_edt -- pinned staging, the int32 -> uint64 conversion and the copies all
inside the timed call.  Usage: python tools/dropin_e2e.py [c1 c2 ...]"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402

CLI = os.path.join(ROOT, "paper_2106_03503_b200", "lib", "dropin_cli")
for cfg in sys.argv[1:] or ["c1", "c2"]:
    img = workloads.config(cfg)
    h, w = img.shape
    with tempfile.TemporaryDirectory() as d:
        fin, fout = os.path.join(d, "in.u8"), os.path.join(d, "out.txt")
        img.tofile(fin)
        subprocess.run([CLI, "time_edt", str(h), str(w), fin, fout, "30"], check=True)
        txt = open(fout).read().split()
    med = float(txt[1])
    print(f"{cfg}: {h}x{w} drop-in edt() host->host median {med:.3f} ms, min {float(txt[3]):.3f} ms, "
          f"{h * w / med / 1e3:.1f} Mpixel/s (uint64 DistanceMap out)")
