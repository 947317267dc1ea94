"""Statistics of the window row pass on a config (CPU model, tuning aid):
segment evaluations per thread, stack sizes.  python tools/win_stats.py c2 [rows]"""
import sys
import numpy as np
sys.path.insert(0, ".")
import workloads

def nearest_rows(feat):
    H, W = feat.shape
    INF = 1 << 20
    up = np.full((H, W), -INF, np.int64)
    last = np.full(W, -INF, np.int64)
    for i in range(H):
        last = np.where(feat[i], i, last); up[i] = last
    dn = np.full((H, W), INF, np.int64)
    nxt = np.full(W, INF, np.int64)
    for i in range(H - 1, -1, -1):
        nxt = np.where(feat[i], i, nxt); dn[i] = nxt
    ii = np.arange(H)[:, None]
    nr = np.where(ii - up <= dn - ii, up, dn)
    return np.where(np.abs(nr) >= INF // 2, -1, nr)

def seg_stack(g, c0, c1, W):
    st = []
    for m in range(c0, c1):
        if g[m] is None: continue
        start = 0
        while st:
            k, s = st[-1]
            num = g[m] - g[k] + m * m - k * k; den = 2 * (m - k)
            if num < s * den: st.pop(); continue
            start = num // den + 1
            break
        if start <= W - 1: st.append((m, start))
    return st

def row_stats(g, W, L):
    nseg = -(-W // L)
    stk = [seg_stack(g, s * L, min(W, s * L + L), W) for s in range(nseg)]
    evals = []; visits = []
    for s in range(nseg):
        c0, cl = s * L, min(L, W - s * L)
        best = [None] * cl
        def ev(st):
            for x in range(cl):
                j = c0 + x
                e = max(e_ for e_ in range(len(st)) if st[e_][1] <= j)
                k = st[e][0]; d = g[k] + (j - k) ** 2
                if best[x] is None or d < best[x]: best[x] = d
        ne = 0; nv = 0
        if stk[s]: ev(stk[s]); ne += 1
        U = max(b if b is not None else 1 << 40 for b in best)
        pl, pr = s - 1, s + 1
        while True:
            while pl >= 0 and not stk[pl]: pl -= 1
            while pr < nseg and not stk[pr]: pr += 1
            gl = c0 - (pl * L + L - 1) if pl >= 0 else None
            gr = pr * L - (c0 + cl - 1) if pr < nseg else None
            okL = gl is not None and gl * gl <= U; okR = gr is not None and gr * gr <= U
            if not okL and not okR: break
            nv += 1
            if okL and (not okR or gl <= gr):
                st = stk[pl]; dx = c0 - st[-1][0]
                if min(g[k] for k, _ in st) + dx * dx <= U: ev(st); ne += 1; U = max(b if b is not None else 1 << 40 for b in best)
                pl -= 1
            else:
                st = stk[pr]; dx = st[0][0] - (c0 + cl - 1)
                if min(g[k] for k, _ in st) + dx * dx <= U: ev(st); ne += 1; U = max(b if b is not None else 1 << 40 for b in best)
                pr += 1
        evals.append(ne); visits.append(nv)
    return evals, [len(x) for x in stk], visits

cfg = sys.argv[1]; nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 16
L = int(sys.argv[3]) if len(sys.argv) > 3 else 32
img = workloads.config(cfg)
if img.ndim == 3: img = img[0]
H, W = img.shape
rng = np.random.default_rng(0)
rows = sorted(rng.choice(H, nrows, replace=False))
for pol in (0, 1):
    feat = (img != 0) if pol == 0 else (img == 0)
    nr = nearest_rows(feat)
    E, S, V = [], [], []
    for i in rows:
        g = [None if nr[i, k] < 0 else int((i - nr[i, k]) ** 2) for k in range(W)]
        e, s, v = row_stats(g, W, L); E += e; S += s; V += v
    E, S, V = np.array(E), np.array(S), np.array(V)
    print(f"{cfg} pol{pol} L={L}: evals/seg mean {E.mean():.2f} p50 {np.median(E):.0f} p90 {np.percentile(E,90):.0f} max {E.max()}; stack mean {S.mean():.2f} max {S.max()}; visits mean {V.mean():.2f} p90 {np.percentile(V,90):.0f}")
