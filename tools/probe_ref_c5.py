"""Probe (GPU box host): cost of the reference CPU path on the FULL c5 image,
and of the C restatement, to size the bench reference arm and parity tests."""
import os, resource, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import workloads
print("cpus", os.cpu_count(), flush=True)
os.system("free -g; nproc; lscpu | grep -E 'Model name|^CPU\\(s\\)|Thread|Socket'")
t = time.time(); img = workloads.config("c5"); print("gen", time.time() - t, int(img.sum()), flush=True)
for th in (os.cpu_count(),):
    t = time.time(); out, ns = oracle.ref_edt(img, threads=th, want_time=True)
    print("ref_edt threads", th, "ns", ns * 1e-9, "wall", time.time() - t, "max", int(out[out != oracle.INF].max()), flush=True)
    del out
print("maxrss GB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, flush=True)
t = time.time(); o2 = oracle.edt(img); print("orc edt wall", time.time() - t, flush=True)
del o2
crop = np.ascontiguousarray(img[:4096, :4096])
t = time.time(); _, ns = oracle.ref_edt(crop, threads=1, want_time=True); print("ref T=1 4096 crop", ns * 1e-9, flush=True)
