"""Danielsson's vector transform (k_vector.cu) against the reference's own
danielsson() on the host: one C1 image (a single warp: the recurrence is
sequential over rows) and a batch of 1024 images of 256^2 (one warp per image).
Output kept as profiles/r02/danielsson.txt."""
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2106_03503_b200 as dfc  # noqa: E402
import workloads  # noqa: E402


def gpu_ms(fn, n=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def cpu_ms(img, n=3):
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        oracle.ref_danielsson(img) if oracle.ref_available() else oracle.danielsson(img)
        ts.append((time.perf_counter() - t) * 1e3)
    return min(ts)


c1 = workloads.config("c1")
d1 = torch.from_numpy(c1).cuda()
g = gpu_ms(lambda: dfc.danielsson(d1))
c = cpu_ms(c1)
print(f"c1 600x500, one image : GPU {g:.3f} ms ({c1.size / g / 1e3:.1f} Mpixel/s), reference on one host thread "
      f"{c:.3f} ms ({c1.size / c / 1e3:.1f} Mpixel/s)")
batch = np.stack([oracle.random_image(256, 256, 0.01, 100 + k) for k in range(1024)])
db = torch.from_numpy(batch).cuda()
g = gpu_ms(lambda: dfc.danielsson(db), n=5)
c = cpu_ms(batch[0]) * 1024
print(f"1024 images of 256x256 : GPU {g:.3f} ms ({batch.size / g / 1e3:.1f} Mpixel/s), reference on one host thread "
      f"~{c:.1f} ms ({batch.size / c / 1e3:.1f} Mpixel/s, 1024 x one image)")
out = dfc.danielsson(db)
torch.cuda.synchronize()
for k in (0, 511, 1023):
    d, dy, dx = oracle.danielsson(batch[k])
    assert (out["sqdist"][k].cpu().numpy().view(np.uint64) == d).all()
print("batch parity ok")
