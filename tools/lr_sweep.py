"""Time the row-pass variants on a config (CUDA events around one edt call,
L2 flushed between calls).  Usage: python tools/lr_sweep.py cfg chunks..."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2106_03503_b200 as dfc
import workloads
cfg = sys.argv[1]
chunks = [int(c) for c in sys.argv[2:]] or [256]
img = torch.from_numpy(workloads.config(cfg)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(fn, reps=10):
    ts = []
    for r in range(reps + 2):
        flush.fill_(r); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(e0.elapsed_time(e1))
    return np.median(ts)
if img.dim() == 3:
    calls = {"batched": lambda: dfc.edt_batched(img, dist=False, label=True)}
else:
    calls = {"pol0": lambda: dfc.edt(img, polarity=0, dist=True), "pol1": lambda: dfc.edt(img, polarity=1, dist=True),
             "dual": lambda: dfc.edt_dual(img)}
ref = {}
for mode in (["default"] if chunks == [0] else ["default", "lr"]):
    dfc.set_row_kernel(mode)
    for ch in ([0] if mode == "default" else chunks):
        dfc.set_lr_chunk(ch)
        res = {k: run(f) for k, f in calls.items()}
        outs = {k: f() for k, f in calls.items()}
        torch.cuda.synchronize()
        if mode == "default":
            ref = outs
            same = "ref"
        else:
            same = all(all(torch.equal(outs[k][q], ref[k][q]) for q in outs[k]) for k in outs)
        print(cfg, mode, ch, {k: round(v, 4) for k, v in res.items()}, "identical" if same else "MISMATCH", flush=True)
