"""Pure-Python model of the streaming row pass (one lane = one row): the
reference stack algorithm (exact_edt.cpp:208-223) scanned left to right with
EAGER FINALISATION -- column F is emitted as soon as no parabola of a later
column can change its owner:

    every future parabola p >= m+1 has D_p(F) >= (p-F)^2 >= (m+1-F)^2, so
    keep_old : D(F) <= (m+1-F)^2  =>  final   (a later column must be strictly smaller)
    take_new : D(F) <  (m+1-F)^2  =>  final   (a later column wins ties)

Only the "live" part of the stack (entries owning columns >= F) is kept, so
the stack stays tiny in practice (<= ~50 entries on the configs).  Output is
a list of runs (start column, owner column) covering [0, W).
Test infrastructure only: mirrors paper_2106_03503_b200/csrc/k_rows_stream.cu.
"""


def stream_row(g, take_new=False, cap=None, emit_cap=None):
    """g: list of squared vertical values or None.  Returns (runs, max_live) where
    runs = [(start_col, k)] ; k = None for a featureless row.  Raises
    OverflowError if the live stack would exceed cap."""
    W = len(g)
    st = []          # live entries [k, start]; st[0] owns column F
    F = 0
    runs = []
    max_live = 0

    def emit(j, k):
        if not runs or runs[-1][1] != k:
            runs.append((j, k))

    def finalize(m):
        nonlocal F
        budget = emit_cap if emit_cap is not None else 1 << 30
        while F <= m and st and budget > 0:
            budget -= 1
            # drop entries whose range ended at or before F
            while len(st) > 1 and st[1][1] <= F:
                st.pop(0)
            k = st[0][0]
            d = g[k] + (F - k) ** 2
            lim = (m + 1 - F) ** 2
            if (d < lim) if take_new else (d <= lim):
                emit(F, k)
                F += 1
            else:
                break

    for m in range(W):
        if g[m] is not None:
            gm = g[m]
            start = None
            while st:
                tk, ts = st[-1]
                num = gm - g[tk] + m * m - tk * tk
                den = 2 * (m - tk)
                if (num <= ts * den) if take_new else (num < ts * den):
                    st.pop()
                    continue
                if (num > (W - 1) * den) if take_new else (num >= (W - 1) * den):
                    start = -1  # never owns a column: skip
                else:
                    q = num // den
                    start = (q + (1 if num != q * den else 0)) if take_new else q + 1
                break
            if start is None:          # stack empty: owns everything not yet final
                start = F
            if start >= 0:
                st.append([m, max(start, F)])
                if cap is not None and len(st) > cap:
                    raise OverflowError
                max_live = max(max_live, len(st))
        finalize(m)
    if not st:
        return [(0, None)], 0
    finalize(W)  # end of row: everything left is final ((W+1-F)^2 > any D)
    while F < W:  # (finalize(W) uses lim >= 1; force the tail)
        while len(st) > 1 and st[1][1] <= F:
            st.pop(0)
        emit(F, st[0][0])
        F += 1
    return runs, max_live


def expand(runs, g, W):
    out = []
    for t, (s, k) in enumerate(runs):
        e = runs[t + 1][0] if t + 1 < len(runs) else W
        for j in range(s, e):
            out.append((None, None) if k is None else (g[k] + (j - k) ** 2, k))
    return out


def stream_chunk(g, c0, c1, s0, take_new=False, cap=None):
    """Chunked streaming (k_rows_stream.cu with chunks): scan candidates from
    s0 (the warm-up start, s0 <= c0), keep the envelope over [F, W) only, F
    starting at c0, emit final columns of [c0, c1) eagerly, scanning past c1
    until they are all final.  Returns (runs over [c0, c1), verified): an
    emitted column is verified when no candidate left of s0 could own it --
    D(F) < (F - s0 + 1)^2 (keep_old; <= for take_new) or s0 == 0."""
    W = len(g)
    st = []                 # live entries [k, start]
    F = c0
    runs = []
    ok = True

    def emit(j, k):
        nonlocal ok
        if k is None:
            if s0 > 0:
                ok = False  # the row may have features left of s0
        else:
            d = g[k] + (j - k) ** 2
            lim = (j - s0 + 1) ** 2
            if s0 > 0 and not ((d <= lim) if take_new else (d < lim)):
                ok = False
        if not runs or runs[-1][1] != k:
            runs.append((j, k))

    def finalize(m1, force=False):
        nonlocal F
        while F < c1 and (force or F < m1):
            if not st:
                if not force:
                    return
                emit(F, None)
                F += 1
                continue
            while len(st) > 1 and st[1][1] <= F:
                st.pop(0)
            k = st[0][0]
            if not force:
                d = g[k] + (F - k) ** 2
                lim = (m1 - F) ** 2
                if not ((d < lim) if take_new else (d <= lim)):
                    return
            emit(F, k)
            F += 1

    for m in range(s0, W):
        if F >= c1:
            break
        if g[m] is not None:
            gm = g[m]
            start = None
            while st:
                tk, ts = st[-1]
                num = gm - g[tk] + m * m - tk * tk
                den = 2 * (m - tk)
                if (num <= ts * den) if take_new else (num < ts * den):
                    st.pop()
                    continue
                if (num > (W - 1) * den) if take_new else (num >= (W - 1) * den):
                    start = -1
                else:
                    q = num // den
                    start = (q + (1 if num != q * den else 0)) if take_new else q + 1
                break
            if start is None:
                start = F
            if start >= 0:
                st.append([m, max(start, F)])
                if cap is not None and len(st) > cap:
                    raise OverflowError
        finalize(m + 1)
    finalize(W, force=True)
    return runs, ok


def chunked_row(g, C, w, take_new=False):
    """Whole row from chunks of C columns, warm-up w, retry with s0 = 0 when a
    chunk fails its verification.  Returns (per-column (D, k), retries)."""
    W = len(g)
    out, retries = [], 0
    for c0 in range(0, W, C):
        c1 = min(c0 + C, W)
        runs, ok = stream_chunk(g, c0, c1, max(0, c0 - w), take_new)
        if not ok:
            retries += 1
            runs, ok = stream_chunk(g, c0, c1, 0, take_new)
            assert ok
        for t, (s, k) in enumerate(runs):
            e = runs[t + 1][0] if t + 1 < len(runs) else c1
            for j in range(s, e):
                out.append((None, None) if k is None else (g[k] + (j - k) ** 2, k))
    return out, retries
