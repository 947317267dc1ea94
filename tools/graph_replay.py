"""Direct launches against a CUDA-graph replay of the same call (the library is
capturable: stream-ordered scratch, event fork/join to its helper stream, no host
synchronisation).  Output kept as profiles/r02/graph_replay.txt."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import paper_2106_03503_b200 as dfc
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in ("c5", "c1", "c2", "c3"):
    img = workloads.config(cfg)
    dev = torch.from_numpy(img).cuda()
    if cfg == "c2":
        out = {k: torch.empty(img.shape, dtype=dt, device="cuda") for k, dt in (("sqdist_bg", torch.int32), ("dist_bg", torch.float32), ("sqdist_obj", torch.int32), ("dist_obj", torch.float32))}
        step = lambda: dfc.edt_dual(dev, out=out)
    elif cfg == "c3":
        out = {k: torch.empty(img.shape, dtype=torch.int32, device="cuda") for k in ("sqdist", "label")}
        step = lambda: dfc.edt_batched(dev, dist=False, label=True, out=out)
    else:
        out = {"sqdist": torch.empty(img.shape, dtype=torch.int32, device="cuda")}
        if cfg == "c1": out["dist"] = torch.empty(img.shape, dtype=torch.float32, device="cuda")
        step = lambda: dfc.edt(dev, dist=cfg == "c1", out=out)
    for _ in range(3): step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.synchronize()
    def timeit(fn, n=20):
        ts = []
        for k in range(n):
            flush.fill_(k & 0xff)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)
    print(cfg, "direct %.4f ms   graph replay %.4f ms" % (timeit(step), timeit(g.replay)))
