"""Pure-Python model of the lane-per-row chunk scan (csrc/k_rows_lr.cu).

One lane owns one row and one column chunk [c0, c1).  It runs the reference's
stack algorithm (exact_edt.cpp:208-223) left to right over the candidates of
[S0, W), with the domain restricted to [c0, c1): starts are clamped to the first column not yet emitted (c0 at first) and a
parabola whose start lies past c1-1 is never pushed (:218 with cols -> c1).

ENTRY-level eager finalisation: after column m has been scanned, every later
parabola p >= m+1 has D_p(j) >= (m+1-j)^2.  The bottom entry (kb, sb) owns
[sb, eb] (eb = next start - 1, or c1-1 for the only entry); its value minus
(m+1-j)^2 is linear and increasing in j, so the entry is final once

    keep_old : g_b + (eb-kb)^2 <= (m+1-eb)^2   (a later column must be strictly smaller)
    take_new : g_b + (eb-kb)^2 <  (m+1-eb)^2   (a later column wins ties)

A final entry is emitted (start, column) and leaves the stack; its range can
no longer change (a later parabola cannot beat it anywhere in [sb, eb], so it
can neither pop it nor start inside it).  The scan stops once the stack is
empty after the chunk's last entry has been emitted.

Bounds: owners are monotone in j under either tie rule, so every owner of
[c0, c1) lies in [owner(c0-1), owner(c1-1)]; only that range is scanned.

Test infrastructure only.
"""


def owner(g, b, take_new=False):
    """Owner of column b (smallest minimising column for keep_old, largest for
    take_new), by the kernel's outward search: stop once the nearest
    unexamined column d has d^2 > best.  None for a featureless row."""
    W = len(g)
    best, bk = None, None
    lo, hi = b, b + 1  # examined [lo, hi)

    def consider(k):
        nonlocal best, bk
        if g[k] is None:
            return
        v = g[k] + (k - b) ** 2
        if best is None or v < best or (v == best and (k > bk if take_new else k < bk)):
            best, bk = v, k

    consider(b)
    while True:
        dl, dr = b - lo + 1, hi - b
        left = lo > 0 and (best is None or dl * dl <= best)
        right = hi < W and (best is None or dr * dr <= best)
        if not (left or right):
            return bk
        if left:
            lo -= 1
            consider(lo)
        if right:
            consider(hi)
            hi += 1


def scan_chunk(g, c0, c1, kS, kE, take_new=False, cap=None):
    """Returns (entries, stats): entries = [(start, k)] covering [c0, c1) in order
    (k None: featureless row), stats = dict(last_m, max_live, pops, pushes)."""
    W = len(g)
    st = []        # live entries [k, start]
    out = []
    F = [c0]       # first column not yet emitted
    stats = dict(max_live=0, pops=0, pushes=0, last_m=kS - 1)

    def floor_div(a, b):
        return a // b

    def try_emit(m):
        # emit final bottom entries after column m was scanned
        while st:
            kb, sb = st[0]
            eb = st[1][1] - 1 if len(st) > 1 else c1 - 1
            d = g[kb] + (eb - kb) ** 2
            lim = (m + 1 - eb) ** 2
            if (d < lim) if take_new else (d <= lim):
                out.append((sb, kb))
                st.pop(0)
                F[0] = eb + 1
                if not st:
                    return True   # chunk complete
            else:
                return False
        return False

    done = False
    for m in range(kS, kE + 1):
        stats["last_m"] = m
        if g[m] is not None:
            gm = g[m]
            push_start = F[0]
            while st:
                tk, ts = st[-1]
                num = gm - g[tk] + m * m - tk * tk
                den = 2 * (m - tk)
                start = -floor_div(-num, den) if take_new else floor_div(num, den) + 1
                if start <= ts:
                    st.pop()
                    stats["pops"] += 1
                    continue
                push_start = start
                break
            if push_start <= c1 - 1:
                st.append([m, max(push_start, F[0])])
                stats["pushes"] += 1
                if cap is not None and len(st) > cap:
                    raise OverflowError
            stats["max_live"] = max(stats["max_live"], len(st))
        if st and try_emit(m):
            done = True
            break
    if not done:
        # end of the row: everything left is final
        while st:
            kb, sb = st.pop(0)
            out.append((sb, kb))
    if not out:
        out.append((c0, None))
    return out, stats


def expand(entries, g, c0, c1):
    """entries -> (D list, owner list) over [c0, c1)."""
    D, K = [], []
    e = 0
    for j in range(c0, c1):
        while e + 1 < len(entries) and entries[e + 1][0] <= j:
            e += 1
        k = entries[e][1]
        if k is None:
            D.append(None)
            K.append(None)
        else:
            D.append(g[k] + (j - k) ** 2)
            K.append(k)
    return D, K


def lr_row(g, C, take_new=False):
    """The whole row by independent chunks; returns (D, owner) lists."""
    W = len(g)
    D, K = [], []
    for c0 in range(0, W, C):
        c1 = min(c0 + C, W)
        kS = owner(g, c0 - 1, take_new) if c0 > 0 else 0
        kE = owner(g, c1 - 1, take_new) if c1 < W else W - 1
        if kS is None or kE is None:  # featureless row
            D += [None] * (c1 - c0)
            K += [None] * (c1 - c0)
            continue
        ent, _ = scan_chunk(g, c0, c1, kS, kE, take_new)
        d, k = expand(ent, g, c0, c1)
        D += d
        K += k
    return D, K
