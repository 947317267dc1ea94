"""Race stand-in (compute-sanitizer racecheck is closed on this pool): every
kernel family on fixed inputs, five runs each with an L2-thrashing kernel in
between, outputs compared bit for bit with the first run and the first run with
the CPU oracle.  A data race on shared or global memory shows up as run-to-run
differences on at least some of these shapes (the cross-warp race fixed in round
1 did)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2106_03503_b200 as dfc  # noqa: E402
import workloads  # noqa: E402

RUNS = 5
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def same(a, b):
    return all(torch.equal(a[k], b[k]) for k in a)


def repeat(name, fn, check=None):
    first = fn()
    torch.cuda.synchronize()
    for r in range(RUNS - 1):
        flush.fill_(r)
        out = fn()
        torch.cuda.synchronize()
        assert same(first, out), f"{name}: run {r + 2} differs from run 1"
    if check is not None:
        check(first)
    print(f"{name}: {RUNS} runs bit-identical" + (", oracle ok" if check else ""))


def main():
    dfc.set_band_min_pixels(0)  # the band path for the small sparse case too
    cases = {
        "anc 1500x2000 p=0.01": workloads.bernoulli(1500, 2000, 0.01, 5),
        "anc discs 2048^2": workloads.discs(2048, 2048, 60, 9),
        "band sparse tiles 4096^2": workloads.sparse_tiles(4096, 4096, tile=256, n_on=64, p=2e-4, seed=3),
        "lr/merge wide 40x20000": workloads.bernoulli(40, 20000, 0.003, 11),
    }
    for name, img in cases.items():
        dev = torch.from_numpy(img).cuda()
        want = oracle.to_i32(oracle.edt(img)) if img.size <= 1 << 23 else None

        def chk(o, want=want):
            if want is not None:
                assert (o["sqdist"].cpu().numpy() == want).all(), "oracle mismatch"
        repeat(name + " (D, dist, label, ncol)", lambda: dfc.edt(dev, dist=True, label=True, nearest_col=True), chk)
        repeat(name + " (D only)", lambda: dfc.edt(dev, dist=False), chk)
        repeat(name + " dual", lambda: dfc.edt_dual(dev))
        repeat(name + " raster", lambda: dfc.raster(dev))
    pts = torch.from_numpy(workloads.points_batch(64, 256, 256, 30, 7)).cuda()
    repeat("pts batch 64x256^2", lambda: dfc.edt_batched(pts, dist=False, label=True))
    many = torch.from_numpy(workloads.points_batch(16, 256, 256, 200, 8)).cuda()
    repeat("batch 16x256^2, 200 points", lambda: dfc.edt_batched(many, dist=True, label=True))
    dn = torch.from_numpy(oracle.random_image(300, 400, 0.02, 6)).cuda()
    repeat("danielsson 300x400", lambda: dfc.danielsson(dn))
    print("determinism ok")


if __name__ == "__main__":
    main()
