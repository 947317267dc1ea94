"""One-polarity EDT of a config image, for profiling: python tools/run_pol.py c2 1 [reps]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_2106_03503_b200 as dfc
import workloads
img = torch.from_numpy(workloads.config(sys.argv[1])).cuda()
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    dfc.edt(img, polarity=int(sys.argv[2]), dist=True)
torch.cuda.synchronize()
print("ok")
