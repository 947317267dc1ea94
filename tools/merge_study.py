"""Offline study of the row-pass merges (tuning aid): how far the takeover
column x lies from the boundary c and from x0, the takeover of the two
parabolas that own c-1 (in A) and c (in B); and how many piece-Newton steps
(x <- takeover of the pieces owning x-1 / x) reach x.
python tools/merge_study.py c2 [rows] [pol]"""
import sys
from collections import Counter

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from row_model import Row
import workloads
sys.path.insert(0, "tools")
from win_stats_lib import nearest_rows  # noqa: E402


def pair_x(a, b, W):
    num = b["g"] - a["g"] + b["k"] ** 2 - a["k"] ** 2
    den = 2 * (b["k"] - a["k"])
    x = num // den + 1  # keep_old: first j with D_b(j) < D_a(j)
    return min(max(x, 0), W)


def main():
    cfg = sys.argv[1]; nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    pol = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    img = workloads.config(cfg)
    if img.ndim == 3: img = img[0]
    H, W = img.shape
    feat = (img != 0) if pol == 0 else (img == 0)
    nr = nearest_rows(feat)
    rng = np.random.default_rng(1)
    L = 32; T = 1
    while T * L < W: T *= 2
    stats = {}
    for i in sorted(rng.choice(H, nrows, replace=False)):
        g = [None if nr[i, k] < 0 else int((i - nr[i, k]) ** 2) for k in range(W)]
        r = Row(g, T, L, False)
        G = 2
        while G <= T:
            half = G // 2
            xs = {}
            for gb in range(0, T, G):
                x = r.probe_merge(gb, gb + half, gb + G, min(G, 32))
                xs[gb] = x
                c = min((gb + half) * L, W - 1)
                a = r.piece_at(gb, gb + half, c - 1); b = r.piece_at(gb + half, gb + G, c)
                st = stats.setdefault(G, Counter())
                if a is None or b is None:
                    st["empty"] += 1; continue
                x0 = pair_x(a, b, W)
                d = abs(x - x0)
                st["x0_exact" if d == 0 else "x0_le2" if d <= 2 else "x0_le32" if d <= 32 else "x0_far"] += 1
                st["c_le32" if abs(x - c) <= 32 else "c_far"] += 1
                # piece-Newton: x <- takeover of the pieces at x-1 (A) / x (B)
                xn, it = x0, 0
                while it < 20:
                    pa = r.piece_at(gb, gb + half, min(max(xn - 1, 0), W - 1))
                    pb = r.piece_at(gb + half, gb + G, min(xn, W - 1))
                    if pa is None or pb is None: break
                    x2 = pair_x(pa, pb, W)
                    it += 1
                    if x2 == xn: break
                    xn = x2
                st["newton_ok" if xn == x else "newton_bad"] += 1
                st[f"newton_it{min(it, 5)}"] += 1
            for s in range(T):
                gb = s & ~(G - 1)
                r.cut[s] = max(r.cut[s], xs[gb]) if (s - gb) >= half else min(r.cut[s], xs[gb])
            G *= 2
    for G in sorted(stats):
        st = stats[G]; n = sum(v for k, v in st.items() if k.startswith("x0") ) or 1
        print(f"G={G:5d}", " ".join(f"{k}={v}" for k, v in sorted(st.items())))




def probe_merge_newton(r, s0, sm, s1, P, newton=True, one_lane=False):
    """k_rows probe search with lanes 0/1 probing the piece-Newton estimate
    (x_n - 1, x_n) instead of uniform positions.  Returns (x, rounds)."""
    W, L = r.W, r.L
    lo, hi = 0, W
    c = min(sm * L, W - 1)
    rounds, xn = 0, None
    while hi > lo:
        n = hi - lo
        ps = []
        for q in range(P):
            if rounds == 0:
                if q < 2: p = c - 1 + q
                elif P >= 4 and q == 2: p = 0
                elif P >= 4 and q == P - 1: p = W - 1
                else: p = lo + ((q - (2 if P >= 4 else 1)) * n) // (P - 3 if P >= 4 else P - 1)
            elif newton and xn is not None and q < (1 if one_lane else 2):
                p = xn - 1 + q if not one_lane else xn
            else:
                nl = (1 if one_lane else 2) if (newton and xn is not None) else 0
                m, qq = P - nl, q - nl
                p = lo + ((qq + 1) * n) // (m + 1)
            ps.append(min(max(p, lo), hi - 1))
        rounds += 1
        bits = [r.beats(s0, sm, s1, p) for p in ps]
        t = min([p for p, b in zip(ps, bits) if b], default=W)
        f = max([p for p, b in zip(ps, bits) if not b], default=-1)
        hi, lo = min(hi, t), max(lo, f + 1)
        # Newton estimate from the pieces at the two leading probes
        if one_lane and rounds > 1:
            pa = r.piece_at(s0, sm, ps[0]); pb = r.piece_at(sm, s1, ps[0])
        else:
            pa = r.piece_at(s0, sm, ps[0]); pb = r.piece_at(sm, s1, ps[1] if P > 1 else ps[0])
        xn = pair_x(pa, pb, W) if (pa is not None and pb is not None) else None
        if xn is not None and not (lo < xn <= hi):
            xn = None
    return lo, rounds


ONE = False


def compare(cfg, nrows, pol):
    img = workloads.config(cfg)
    if img.ndim == 3: img = img[0]
    H, W = img.shape
    nr = nearest_rows((img != 0) if pol == 0 else (img == 0))
    rng = np.random.default_rng(1)
    L = 32; T = 1
    while T * L < W: T *= 2
    tot = {}
    for i in sorted(rng.choice(H, nrows, replace=False)):
        g = [None if nr[i, k] < 0 else int((i - nr[i, k]) ** 2) for k in range(W)]
        r = Row(g, T, L, False)
        G = 2
        while G <= T:
            half, P = G // 2, min(G, 32)
            xs, rs = {}, {}
            for gb in range(0, T, G):
                x0, r0 = probe_merge_newton(r, gb, gb + half, gb + G, P, newton=False)
                x1, r1 = probe_merge_newton(r, gb, gb + half, gb + G, P, newton=True, one_lane=ONE)
                assert x0 == x1, (G, gb, x0, x1)
                xs[gb] = x0; rs[gb] = (r0, r1)
            # warp cost = max rounds over the merges sharing a warp (32 lanes)
            per_warp = max(1, 32 // G) if G <= 32 else 1
            keys = sorted(rs)
            a = tot.setdefault(G, [0, 0, 0, 0])
            for w in range(0, len(keys), per_warp):
                grp = keys[w:w + per_warp]
                a[0] += max(rs[k][0] for k in grp); a[1] += max(rs[k][1] for k in grp)
                a[2] += sum(rs[k][0] for k in grp); a[3] += sum(rs[k][1] for k in grp)
            for s in range(T):
                gb = s & ~(G - 1)
                r.cut[s] = max(r.cut[s], xs[gb]) if (s - gb) >= half else min(r.cut[s], xs[gb])
            G *= 2
    for G in sorted(tot):
        a = tot[G]
        print(f"G={G:5d} warp-rounds probe {a[0]:5d} newton {a[1]:5d} | merge-rounds probe {a[2]:5d} newton {a[3]:5d}")


if __name__ == "__main__":
    if len(sys.argv) > 4 and sys.argv[4] == "compare":
        ONE = len(sys.argv) > 5
        compare(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
    else:
        main()
