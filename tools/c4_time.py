"""Time dfc.raster on config 4 (CUDA events, L2 flushed between calls) and check
the three maps against the default build.  python tools/c4_time.py"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2106_03503_b200 as dfc
import workloads
img = torch.from_numpy(workloads.config("c4")).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for r in range(12):
    flush.fill_(r); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); out = dfc.raster(img); e1.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(e0.elapsed_time(e1))
h = {k: int(torch.sum(v.to(torch.int64) * (torch.arange(v.numel(), device=v.device).view(v.shape) % 9973 + 1)).item()) for k, v in out.items()}
print("c4 raster ms", round(float(np.median(ts)), 4), h)
