"""Time the column pass and row pass separately (CUDA events via the profile hook)
for a config, per polarity.  Usage: python tools/time_parts.py c2 [reps]"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2106_03503_b200 as dfc
import workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
img = torch.from_numpy(workloads.config(cfg)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

def timeit(fn):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for x in e:
        x.record()
    col, row = [], []
    for r in range(reps + 2):
        flush.fill_(r)
        dfc.set_profile_events(*e)
        fn()
        torch.cuda.synchronize()
        if r >= 2:
            col.append(e[0].elapsed_time(e[1])); row.append(e[1].elapsed_time(e[2]))
    dfc.set_profile_events(None, None, None)
    return np.median(col), np.median(row)

if img.dim() == 2:
    for pol in (0, 1):
        c, r = timeit(lambda: dfc.edt(img, polarity=pol, dist=True))
        print(f"{cfg} polarity {pol}: column pass {c:.3f} ms, row pass {r:.3f} ms")
    c, r = timeit(lambda: dfc.edt_dual(img))
    print(f"{cfg} dual: column pass {c:.3f} ms, row pass {r:.3f} ms")
else:
    c, r = timeit(lambda: dfc.edt_batched(img, dist=False, label=True))
    print(f"{cfg} batched: column pass {c:.3f} ms, row pass {r:.3f} ms")
