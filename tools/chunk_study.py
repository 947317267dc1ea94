"""Work of the chunked streaming row pass on a config (tuning aid): columns
scanned per output column (warm-up + chunk + look-ahead), retry rate, live
stack size.  python tools/chunk_study.py c2 rows pol C w"""
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tools")
import stream_model as sm
import workloads
from win_stats_lib import nearest_rows


def scan_len(g, c0, c1, s0, tn):
    """columns scanned until [c0, c1) is final (re-run of stream_chunk's loop)."""
    W = len(g)
    # bisection on the stop column is overkill; emulate by running with growing W cut
    runs, ok = sm.stream_chunk(g, c0, c1, s0, tn)
    # find the smallest m_end such that stream_chunk over g[:m_end] padded with None gives same runs
    lo, hi = c1, W
    while lo < hi:
        mid = (lo + hi) // 2
        g2 = g[:mid] + [None] * (W - mid)
        r2, _ = sm.stream_chunk(g2, c0, c1, s0, tn)
        if r2 == runs:
            hi = mid
        else:
            lo = mid + 1
    return lo - s0, ok


cfg, nrows, pol, C, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
img = workloads.config(cfg)
if img.ndim == 3: img = img[0]
H, W = img.shape
nr = nearest_rows((img != 0) if pol == 0 else (img == 0))
rng = np.random.default_rng(2)
scanned = out = fails = chunks = 0
for i in sorted(rng.choice(H, nrows, replace=False)):
    g = [None if nr[i, k] < 0 else int((i - nr[i, k]) ** 2) for k in range(W)]
    for c0 in range(0, W, C):
        c1 = min(c0 + C, W)
        n, ok = scan_len(g, c0, c1, max(0, c0 - w), False)
        chunks += 1; out += c1 - c0
        scanned += n
        if not ok:
            fails += 1
            n2, _ = scan_len(g, c0, c1, 0, False)
            scanned += n2
print(f"{cfg} pol{pol} C={C} w={w}: scanned/output {scanned/out:.2f}, chunk retries {fails}/{chunks}")


def bound_s0(g, c0, c1):
    """warm-up start from the chunk's own candidates: b(F) = min_F' a_F' + |F - F'|
    >= sqrt(D(F)); s0 = max(0, min_F (F - b(F))); 0 if the chunk has none."""
    INF = 1 << 40
    a = [INF if g[k] is None else int(round(g[k] ** 0.5)) for k in range(c0, c1)]
    n = len(a); b = a[:]
    for x in range(1, n): b[x] = min(b[x], b[x - 1] + 1)
    for x in range(n - 2, -1, -1): b[x] = min(b[x], b[x + 1] + 1)
    if b[0] >= INF: return 0
    return max(0, min(c0 + x - b[x] for x in range(n)))


if len(sys.argv) > 6 and sys.argv[6] == "bound":
    scanned = out = fails = 0
    for i in sorted(rng.choice(H, nrows, replace=False)):
        g = [None if nr[i, k] < 0 else int((i - nr[i, k]) ** 2) for k in range(W)]
        for c0 in range(0, W, C):
            c1 = min(c0 + C, W)
            s0 = bound_s0(g, c0, c1)
            n, ok = scan_len(g, c0, c1, s0, False)
            out += c1 - c0; scanned += n; fails += (not ok)
    print(f"{cfg} pol{pol} C={C} bound warm-up: scanned/output {scanned/out:.2f}, failures {fails}")
