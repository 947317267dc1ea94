"""Pure-Python model of the anchored-segment row pass (csrc/k_rows_anc.cu).

Row of W columns, vertical values g_k (None: no object in column k).  The
kernel works on h_k = g_k + k^2 (kAncInf + k^2 for None) and compares
D_k(j) - j^2 = h_k - 2jk.

  anchors   owner(L s) for every segment s (L = 32 in the kernel), by levels
            of a divide and conquer over the segment index: owner(L s) lies in
            [owner(L s_lo), owner(L s_hi)] for computed s_lo < s < s_hi; the
            bounds are the row ends (a range holding None columns still holds
            its finite owner, which beats them).  An object pixel ON the row
            (g = 0) owns itself.  Owner = smallest minimiser (keep_old) or
            largest (take_new); the kernel scans lane-strided and reduces.
  segments  column j of [L s, L s + L): minimum over the candidates
            [owner(L s), owner(L s + L)] (owner(W) := W - 1), ascending, keep_old
            updating on <, take_new on <=; the value-only path scans the
            aligned superset [lo & ~3, hi | 3] (extra candidates cannot go below
            the minimum the range attains).

Test infrastructure only.
"""

INF = 40000 * 40000  # kAncInf


def _h(g):
    return [(INF if v is None else v) + k * k for k, v in enumerate(g)]


def owner_in(h, j, lo, hi, take_new):
    best, bk = None, None
    for k in range(lo, hi + 1):
        v = h[k] - 2 * j * k
        if best is None or v < best or (take_new and v == best):
            best, bk = v, k
    return bk


def anc_row(g, take_new=False, L=32, superset=False):
    """(D list, owner list) as the kernel computes them; (None, None) entries for a
    featureless row."""
    W = len(g)
    if all(v is None for v in g):
        return [None] * W, [None] * W
    h = _h(g) + [INF + k * k for k in range(W, W + 4)]
    S = (W + L - 1) // L
    P = 1
    while P < S:
        P <<= 1
    anc = [None] * (S + 1)
    anc[S] = W - 1
    step = P >> 1
    while step >= 1:
        for s in range(step, S, 2 * step):
            j = L * s
            if g[j] == 0:
                anc[s] = j
                continue
            lo = 0 if s - step == 0 else anc[s - step]
            hi = W - 1 if s + step >= S else anc[s + step]
            anc[s] = owner_in(h, j, lo, hi, take_new)
        step >>= 1
    anc[0] = 0 if g[0] == 0 else owner_in(h, 0, 0, anc[1] if S > 1 else W - 1, take_new)
    D, K = [], []
    for s in range(S):
        lo, hi = anc[s], anc[s + 1]
        if superset:
            lo, hi = lo & ~3, min(hi | 3, len(h) - 1)
        for j in range(L * s, min(L * s + L, W)):
            k = owner_in(h, j, lo, hi, take_new)
            D.append(h[k] - 2 * j * k + j * j)
            K.append(k)
    return D, K
