"""One C2 edt call with the "lr" row kernel (for ncu captures).
Usage: python tools/lr_one.py [polarity] [chunk] [mode]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_03503_b200 as dfc
import workloads

pol = int(sys.argv[1]) if len(sys.argv) > 1 else 0
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 512
mode = sys.argv[3] if len(sys.argv) > 3 else "lr"
cfg = sys.argv[4] if len(sys.argv) > 4 else "c2"
img = torch.from_numpy(workloads.config(cfg)).cuda()
dfc.set_row_kernel(mode)
dfc.set_lr_chunk(chunk)
for _ in range(3):
    if img.dim() == 3:
        out = dfc.edt_batched(img, dist=False, label=True)
    else:
        out = dfc.edt(img, polarity=pol, dist=cfg != "c5")  # c5: squared distances only
torch.cuda.synchronize()
print("ok")
