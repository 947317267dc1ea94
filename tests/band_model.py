"""Pure-Python model of the band-candidate row pass for sparse planes
(csrc/k_rows_band.cu): k_hull (hull filter) + k_band_rows + k_rows_fill.

Test infrastructure only; statement-level mirror of the kernels, fuzzed
against brute force in tests/test_band_model.py.

Setting: a plane of H x W pixels cut into bands of 32 rows.  For band b
(rows i0 = 32 b .. i1 = min(32 b + 31, H - 1)) the column pass provides, per
column k, the nearest object row ABOVE the band (carry `above`) and BELOW it
(carry `below`), plus the band's own 32-bit mask.

Candidate filter (k_band_hull).  The owner of pixel (i, j), i in the band, is
a nearest object pixel s* = (r*, k*).
  * r* < i0: s* is also the nearest among the objects above the band, so (by
    convexity of its Voronoi cell among those objects, which contains s* in
    its interior) its cell crosses the line i = i0, and s* is the carry above
    of column k*.  Hence the parabola (i0 - above_k*)^2 + (x - k*)^2 touches
    the lower envelope (over REAL x) of the band's above-carry parabolas at
    line i0: the point (k*, H_k*), H_k = (i0 - above_k)^2 + k^2, lies on the
    lower convex hull of those points (collinear points kept: ties).
  * r* > i1: the same with the below carries at line i1.
  * otherwise column k* holds an object pixel inside the band.
So the candidate columns of the band are: the vertices (and collinear points)
of the two lower hulls, plus every column with an object in the band.  Any
superset works (the row pass evaluates the true g_k(i) of every candidate),
so the kernel computes the hulls per WINDOW of 32 x 32 columns (a global hull
point is on the hull of every subset holding it): lane = 32 columns, a
monotone chain with the stack as a 32-bit mask, then 5 levels of pairwise
bridge merges (walk the lower common tangent) inside the warp.

Row pass (k_band_rows).  Lane = row of the band; every lane runs the
reference's stack algorithm (exact_edt.cpp:208-223, integer boundaries,
keep_old / take_new) over the band's candidate columns in ascending order,
with g_k(i) from the band mask and the carries (the upper row on ties,
exact_edt.cpp:351).  The stack's top kCap entries live in a shared-memory
ring; a full ring spills its bottom entry to the row's list in global memory
and an emptied ring reloads the list's last entry, so the stack is unbounded
and no row needs a fallback.  The final stack IS the row's owner list
(column | start << 16, plus the column's nearest row).

Fill (k_rows_fill): lane = column, walk the list (lr_fill_row).
"""

KNOROW = None


def carries(img, H, W):
    """above[b][k], below[b][k] (None = no object) and masks[b][k] (bit r = row 32b+r)."""
    nb = (H + 31) // 32
    above = [[None] * W for _ in range(nb)]
    below = [[None] * W for _ in range(nb)]
    masks = [[0] * W for _ in range(nb)]
    for b in range(nb):
        for k in range(W):
            m = 0
            for r in range(32 * b, min(32 * b + 32, H)):
                if img[r][k]:
                    m |= 1 << (r - 32 * b)
            masks[b][k] = m
    for k in range(W):
        last = None
        for b in range(nb):
            above[b][k] = last
            for r in range(32 * b, min(32 * b + 32, H)):
                if img[r][k]:
                    last = r
        nxt = None
        for b in range(nb - 1, -1, -1):
            below[b][k] = nxt
            for r in range(min(32 * b + 31, H - 1), 32 * b - 1, -1):
                if img[r][k]:
                    nxt = r
    return above, below, masks


def _strictly_above(ka, Ha, kb, Hb, kc, Hc):
    """point b strictly above the segment a-c (ka < kb < kc)."""
    return (Hb - Ha) * (kc - kb) > (Hc - Hb) * (kb - ka)


def window_hull(car, line, w0, lane_cols=32, lanes=32, W=None, cap=None):
    """Candidate columns of one group of `lanes` lanes x `lane_cols` columns
    starting at w0 (k_band_hull: lane = a window of the row, the group = the
    whole row): per-lane monotone chains, then log2(lanes) levels of bridge
    merges.  A lane whose stack would exceed `cap` entries contributes all its
    valid columns and sits out the merges (a superset: a hull point of the row
    is a hull point of every subset holding it)."""
    W = len(car) if W is None else W

    def Hof(k):
        d = line - car[k] if car[k] <= line else car[k] - line
        return d * d + k * k

    def valid(k):
        return k < W and car[k] is not None

    # lane-local hulls: bit c of hm[l] = column w0 + lane_cols*l + c
    hm = [0] * lanes
    overflow = set()
    for l in range(lanes):
        st = []
        for c in range(lane_cols):
            k = w0 + lane_cols * l + c
            if not valid(k):
                continue
            while len(st) >= 2:
                a, bb = st[-2], st[-1]
                if _strictly_above(a, Hof(a), bb, Hof(bb), k, Hof(k)):
                    st.pop()
                else:
                    break
            if cap is not None and len(st) == cap:
                for c2 in range(lane_cols):
                    if valid(w0 + lane_cols * l + c2):
                        overflow.add(w0 + lane_cols * l + c2)
                st = []
                break
            st.append(k)
        for k in st:
            hm[l] |= 1 << (k - w0 - lane_cols * l)

    def col(l, c):
        return w0 + lane_cols * l + c

    def pred(x, glo):  # previous hull column < x in lanes [glo, lane(x)]
        l, c = divmod(x - w0, lane_cols)
        m = hm[l] & ((1 << c) - 1)
        while m == 0 and l > glo:
            l -= 1
            m = hm[l]
        return -1 if m == 0 else col(l, m.bit_length() - 1)

    def succ(x, ghi):  # next hull column > x in lanes [lane(x), ghi)
        l, c = divmod(x - w0, lane_cols)
        m = hm[l] & ~((1 << (c + 1)) - 1)
        while m == 0 and l < ghi - 1:
            l += 1
            m = hm[l]
        return -1 if m == 0 else col(l, (m & -m).bit_length() - 1)

    def clear(x):
        l, c = divmod(x - w0, lane_cols)
        hm[l] &= ~(1 << c)

    g = 1
    while g < lanes:
        for lead in range(0, lanes, 2 * g):
            mid, end = lead + g, lead + 2 * g
            # a = last hull column of the left group, b = first of the right
            a = -1
            for l in range(mid - 1, lead - 1, -1):
                if hm[l]:
                    a = col(l, hm[l].bit_length() - 1)
                    break
            b = -1
            for l in range(mid, end):
                if hm[l]:
                    b = col(l, (hm[l] & -hm[l]).bit_length() - 1)
                    break
            if a < 0 or b < 0:
                continue
            while True:
                moved = False
                while True:
                    p = pred(a, lead)
                    if p >= 0 and _strictly_above(p, Hof(p), a, Hof(a), b, Hof(b)):
                        clear(a)
                        a = p
                        moved = True
                    else:
                        break
                while True:
                    s = succ(b, end)
                    if s >= 0 and _strictly_above(a, Hof(a), b, Hof(b), s, Hof(s)):
                        clear(b)
                        b = s
                        moved = True
                    else:
                        break
                if not moved:
                    break
        g *= 2
    out = set(overflow)
    for l in range(lanes):
        for c in range(lane_cols):
            if (hm[l] >> c) & 1:
                out.add(col(l, c))
    return out


def list_prune(pts, rounds=10, strides=(1, 2, 4, 8, 16, 32, 64)):
    """warp_prune (k_rows_band.cu): a compact ascending point list [(k, H)]
    pruned towards its lower hull.  Each round marks point i when it lies
    strictly above the chord of its list neighbours i - s and i + s for some
    stride s (all marks from the same snapshot), then compacts the survivors.
    Returns the surviving columns: a superset of the hull, collinear points
    kept."""
    col = [p[0] for p in pts]
    Hh = [p[1] for p in pts]
    for _ in range(rounds):
        n = len(col)
        if n < 3:
            break
        gone = [False] * n
        for i in range(n):
            for s in strides:
                if i >= s and i + s < n and _strictly_above(col[i - s], Hh[i - s], col[i], Hh[i], col[i + s], Hh[i + s]):
                    gone[i] = True
        if not any(gone):
            break
        col = [c for c, g in zip(col, gone) if not g]
        Hh = [h for h, g in zip(Hh, gone) if not g]
    return set(col)


def hier_group_candidates(above, below, masks, g0, g1, cb0, cb1, H, W, lanes=32, win=None, cap=None):
    """The candidate columns of bands g0..g1 (a group) inside the coarse group
    cb0..cb1, as k_hull<0/1/2> compute them: filters (list_prune) at the coarse
    lines over all columns (per window of `win` columns, then over the windows'
    survivors), then at the group's line over the coarse survivors plus the
    object columns in between; plus the group's own object columns.  A list
    longer than `cap` is passed through unfiltered.  `lanes` = prune rounds."""
    win = W if win is None else win

    def hull_of(cols, car, line):
        cols = sorted(c for c in cols if car[c] is not None)
        if cap is not None and len(cols) > cap:
            return set(cols)
        return list_prune([(k, (line - car[k]) ** 2 + k * k) for k in cols], rounds=lanes)

    def objcols(b0, b1):
        return set(k for bb in range(b0, b1 + 1) for k in range(W) if masks[bb][k])

    out = objcols(g0, g1)
    for side in (0, 1):
        ckb = cb1 if side else cb0
        car_c = below[ckb] if side else above[ckb]
        cline = min(32 * ckb + 31, H - 1) if side else 32 * ckb
        wins = set()
        for w0 in range(0, W, win):
            wins |= hull_of(range(w0, min(W, w0 + win)), car_c, cline)
        coarse = hull_of(wins, car_c, cline)
        gkb = g1 if side else g0
        car_g = below[gkb] if side else above[gkb]
        gline = min(32 * gkb + 31, H - 1) if side else 32 * gkb
        if (side == 0 and g0 == cb0) or (side == 1 and g1 == cb1):
            out |= coarse
        else:
            between = objcols(g1 + 1, cb1) if side else objcols(cb0, g0 - 1)
            out |= hull_of(coarse | between, car_g, gline)
    return out


def band_candidates(above, below, masks, b, H, W, lane_cols=32, lanes=32, hcap=None):
    i0, i1 = 32 * b, min(32 * b + 31, H - 1)
    cand = set(k for k in range(W) if masks[b][k])
    win = lane_cols * lanes
    for w0 in range(0, W, win):
        cand |= window_hull(above[b], i0, w0, lane_cols, lanes, W, hcap)
        cand |= window_hull(below[b], i1, w0, lane_cols, lanes, W, hcap)
    return sorted(cand)


def nearest_row(i, b, m, ca, cb):
    """Nearest object row of a column for row i of band b (upper on ties)."""
    r0 = 32 * b
    br = i - r0
    up = m & ((1 << (br + 1)) - 1)
    dn = m >> br
    ra = r0 + up.bit_length() - 1 if up else ca
    rb = i + ((dn & -dn).bit_length() - 1) if dn else cb
    if ra is None:
        return rb
    if rb is None:
        return ra
    return ra if i - ra <= rb - i else rb


def row_stack(i, b, cand, above, below, masks, W, take_new, cap=32):
    """One lane's stack over the band's candidates with a `cap`-entry ring that
    spills its bottom to the global list and reloads from it.  Returns the list
    [(k, start, r)] (start increasing from 0)."""
    gl = []       # global list (spilled bottom of the stack)
    ring = []     # top entries (ring[-1] = top)
    stats = {"spills": 0, "reloads": 0}
    for m in cand:
        r = nearest_row(i, b, masks[b][m], above[b][m], below[b][m])
        if r is None:
            continue
        gm = (i - r) ** 2
        start = 0
        push = True
        while True:
            if not ring:
                if not gl:
                    break
                ring.append(gl.pop())
                stats["reloads"] += 1
            tk, ts, tr = ring[-1]
            tg = (i - tr) ** 2
            dm = m - tk
            num = gm - tg + dm * (m + tk)
            den = 2 * dm
            lim = ts * den
            if (num <= lim) if take_new else (num < lim):
                ring.pop()
                continue
            if (num > (W - 1) * den) if take_new else (num >= (W - 1) * den):
                push = False
                break
            q = num // den
            start = (q + (1 if num != q * den else 0)) if take_new else q + 1
            break
        if not push:
            continue
        if len(ring) == cap:
            gl.append(ring.pop(0))
            stats["spills"] += 1
        ring.append((m, start, r))
    gl.extend(ring)
    return gl, stats


def owner_of(i, b, cand, above, below, masks, x, take_new):
    """Exact owner (column) of column x of row i among the candidates (None: no
    finite candidate) -- k_band_rows' outward search."""
    best, bk = None, None
    for m in cand:
        r = nearest_row(i, b, masks[b][m], above[b][m], below[b][m])
        if r is None:
            continue
        v = (i - r) ** 2 + (x - m) ** 2
        if best is None or v < best or (v == best and (m > bk if take_new else m < bk)):
            best, bk = v, m
    return bk


def row_stack_chunked(i, b, cand, above, below, masks, W, take_new, nch=8, cap=16):
    """k_band_rows: the candidates cut into nch chunks of equal counts, chunk w
    = columns [c0, c1) from the 32-column block of its first candidate; each
    chunk runs the stack over [owner(c0-1), owner(c1-1)] with the domain
    restricted to [c0, c1).  Returns [(c0, c1, list)]."""
    n = len(cand)
    out = []
    bounds = []
    for w in range(nch):
        ilo, ihi = w * n // nch, (w + 1) * n // nch
        c0 = 0 if w == 0 else (W if ilo >= n else cand[ilo] & ~31)
        c1 = W if (w == nch - 1 or ihi >= n) else cand[ihi] & ~31
        bounds.append((c0, c1))
    for (c0, c1) in bounds:
        if c0 >= c1:
            continue
        kS = owner_of(i, b, cand, above, below, masks, c0 - 1, take_new) if c0 > 0 else (cand[0] if cand else None)
        kE = owner_of(i, b, cand, above, below, masks, c1 - 1, take_new) if c1 < W else (cand[-1] if cand else None)
        sub = [] if kS is None else [m for m in cand if kS <= m <= kE]
        gl, ring = [], []
        for m in sub:
            r = nearest_row(i, b, masks[b][m], above[b][m], below[b][m])
            if r is None:
                continue
            gm = (i - r) ** 2
            start, push = c0, True
            while True:
                if not ring:
                    if not gl:
                        break
                    ring.append(gl.pop())
                tk, ts, tr = ring[-1]
                dm = m - tk
                num = gm - (i - tr) ** 2 + dm * (m + tk)
                den = 2 * dm
                if (num <= ts * den) if take_new else (num < ts * den):
                    ring.pop()
                    continue
                if (num > (c1 - 1) * den) if take_new else (num >= (c1 - 1) * den):
                    push = False
                    break
                q = num // den
                start = (q + (1 if num != q * den else 0)) if take_new else q + 1
                break
            if not push:
                continue
            if len(ring) == cap:
                gl.append(ring.pop(0))
            ring.append((m, start, r))
        gl.extend(ring)
        out.append((c0, c1, gl))
    return out


def fill(lst, i, W):
    """D and owner per column from a row list (None for a featureless row)."""
    if not lst:
        return [None] * W, [None] * W, [None] * W
    D, K, R = [], [], []
    e = 0
    for j in range(W):
        while e + 1 < len(lst) and lst[e + 1][1] <= j:
            e += 1
        k, _, r = lst[e]
        D.append((i - r) ** 2 + (j - k) ** 2)
        K.append(k)
        R.append(r)
    return D, K, R


def band_transform_chunked(img, take_new=False, nch=8, cap=16, group=1, coarse=None, lanes=32, win=None, hcap=None):
    """(D, K, R) via grouped candidates (k_band_hull: hullA of the group's first
    band + hullB of its last + the group's object columns) and chunked stacks."""
    H, W = len(img), len(img[0])
    above, below, masks = carries(img, H, W)
    nb = (H + 31) // 32
    Dm, Km, Rm = [], [], []
    for b in range(nb):
        g0 = b // group * group
        g1 = min(nb - 1, g0 + group - 1)
        cand = set()
        if coarse is not None:  # k_hull: coarse lines, then the group's lines
            cb0 = g0 // coarse * coarse
            cand = hier_group_candidates(above, below, masks, g0, g1, cb0, min(nb - 1, cb0 + coarse - 1), H, W,
                                         lanes, win, hcap)
        else:
            for bb in range(g0, g1 + 1):
                cand |= set(k for k in range(W) if masks[bb][k])
            cand |= window_hull(above[g0], 32 * g0, 0, W, 1, W)
            cand |= window_hull(below[g1], min(32 * g1 + 31, H - 1), 0, W, 1, W)
        cand = sorted(cand)
        for i in range(32 * b, min(32 * b + 32, H)):
            D, K, R = [None] * W, [None] * W, [None] * W
            for (c0, c1, lst) in row_stack_chunked(i, b, cand, above, below, masks, W, take_new, nch, cap):
                if not lst:
                    continue
                e = 0
                for j in range(c0, c1):
                    while e + 1 < len(lst) and lst[e + 1][1] <= j:
                        e += 1
                    k, _, r = lst[e]
                    D[j], K[j], R[j] = (i - r) ** 2 + (j - k) ** 2, k, r
            Dm.append(D)
            Km.append(K)
            Rm.append(R)
    return Dm, Km, Rm


def band_transform(img, take_new=False, cap=32, lane_cols=32, lanes=32, hcap=None):
    """(D, K, R) maps of a plane via the band path; stats per row."""
    H, W = len(img), len(img[0])
    above, below, masks = carries(img, H, W)
    Dm, Km, Rm = [], [], []
    ncand = []
    st_all = {"spills": 0, "reloads": 0}
    for b in range((H + 31) // 32):
        cand = band_candidates(above, below, masks, b, H, W, lane_cols, lanes, hcap)
        ncand.append(len(cand))
        for i in range(32 * b, min(32 * b + 32, H)):
            lst, st = row_stack(i, b, cand, above, below, masks, W, take_new, cap)
            for key in st_all:
                st_all[key] += st[key]
            D, K, R = fill(lst, i, W)
            Dm.append(D)
            Km.append(K)
            Rm.append(R)
    return Dm, Km, Rm, ncand, st_all


def brute(img, take_new=False):
    """Per pixel: (D, owner column, owner row) with the reference's tie rules:
    keep_old -> smallest minimising column, upper row; take_new -> largest
    minimising column (its upper row)."""
    H, W = len(img), len(img[0])
    sites = [(r, k) for r in range(H) for k in range(W) if img[r][k]]
    Dm, Km, Rm = [], [], []
    for i in range(H):
        D, K, R = [], [], []
        for j in range(W):
            if not sites:
                D.append(None)
                K.append(None)
                R.append(None)
                continue
            best = min((i - r) ** 2 + (j - k) ** 2 for r, k in sites)
            mins = [(k, r) for r, k in sites if (i - r) ** 2 + (j - k) ** 2 == best]
            k = max(x[0] for x in mins) if take_new else min(x[0] for x in mins)
            r = min(x[1] for x in mins if x[0] == k)
            D.append(best)
            K.append(k)
            R.append(r)
        Dm.append(D)
        Km.append(K)
        Rm.append(R)
    return Dm, Km, Rm
