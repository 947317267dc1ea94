"""Does running the two C2 polarities concurrently (two streams) beat running
them back to back?  python tools/overlap_test.py"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2106_03503_b200 as dfc
import workloads
img = torch.from_numpy(workloads.config("c2")).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def seq():
    dfc.edt(img, polarity=0, dist=True); dfc.edt(img, polarity=1, dist=True)
def par():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        dfc.edt(img, polarity=0, dist=True)
    with torch.cuda.stream(s2):
        dfc.edt(img, polarity=1, dist=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
def dual():
    dfc.edt_dual(img)
for name, fn in [("seq", seq), ("par", par), ("dual", dual), ("par", par), ("seq", seq)]:
    ts = []
    for r in range(14):
        flush.fill_(r); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r >= 4: ts.append(e0.elapsed_time(e1))
    print(name, round(float(np.median(ts)), 4), flush=True)
