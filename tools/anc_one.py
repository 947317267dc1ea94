"""Run one config's row pass a few times under a chosen row kernel (for ncu).
Usage: DFC_ROWS=anc python tools/anc_one.py c2 [polarity|dual] [reps]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_03503_b200 as dfc
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "0"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
img = torch.from_numpy(workloads.config(cfg)).cuda()
for _ in range(reps):
    if mode == "dual":
        dfc.edt_dual(img)
    else:
        dfc.edt(img, polarity=int(mode), dist=True)
torch.cuda.synchronize()
print("ok")
