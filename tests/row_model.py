"""Pure-Python model of the k_rows algorithm (segment stacks + leader-walk merges
+ fill), statement for statement, for CPU testing of the merge logic.
Test infrastructure only."""
INF = None


def floor_div(a, b):
    return a // b


def build_segment(g, c0, c1, W, take_new):
    """Stack of (k, start) for columns [c0, c1) over the domain [0, W)."""
    st = []
    for m in range(c0, c1):
        if g[m] is None:
            continue
        num = den = None
        while st:
            tk, ts = st[-1]
            num = g[m] - g[tk] + m * m - tk * tk
            den = 2 * (m - tk)
            lim = ts * den
            pop = num <= lim if take_new else num < lim
            if not pop:
                break
            st.pop()
        start = 0
        if st:
            lim = (W - 1) * den
            if (num > lim) if take_new else (num >= lim):
                continue
            q = num // den
            start = (q + (1 if num != q * den else 0)) if take_new else q + 1
        st.append((m, start))
    return st


class Row:
    def __init__(self, g, T, L, take_new):
        self.g, self.T, self.L, self.W, self.tn = g, T, L, len(g), take_new
        self.stk = [build_segment(g, s * L, min(s * L + L, self.W), self.W, take_new) for s in range(T)]
        self.cut = [0] * T
        self.stats = []

    def owner(self, s0, s1, j):
        lo, hi = s0, s1 - 1
        while lo < hi:
            mid = (lo + hi + 1) >> 1
            if self.cut[mid] <= j:
                lo = mid
            else:
                hi = mid - 1
        return lo

    def entry(self, s, j):
        st = self.stk[s]
        lo, hi = 0, len(st) - 1
        while lo < hi:
            mid = (lo + hi + 1) >> 1
            if st[mid][1] <= j:
                lo = mid
            else:
                hi = mid - 1
        return lo

    def make_piece(self, s, e, s1):
        st = self.stk[s]
        k, start = st[e]
        seg_hi = self.cut[s + 1] if s + 1 < s1 else self.W
        lo = max(start, self.cut[s])
        hi = min(st[e + 1][1] if e + 1 < len(st) else self.W, seg_hi)
        return dict(s=s, e=e, k=k, g=self.g[k], lo=lo, hi=hi)

    def piece_at(self, s0, s1, j):
        s = self.owner(s0, s1, j)
        if not self.stk[s]:
            return None
        return self.make_piece(s, self.entry(s, j), s1)

    def takeover(self, s0, sm, s1, max_steps=100000):
        W, L, tn = self.W, self.L, self.tn
        p0 = min(sm * L, W - 1)
        b = self.piece_at(sm, s1, p0)
        if b is None:
            return W
        a = self.piece_at(s0, sm, p0)
        if a is None:
            return 0
        moved = 0  # -1 after a step left (pred true at the old lo), +1 after a step right
        for _ in range(max_steps):
            lo, hi = max(a["lo"], b["lo"]), min(a["hi"], b["hi"])
            assert lo < hi, (a, b)
            num = b["g"] - a["g"] + b["k"] ** 2 - a["k"] ** 2
            den = 2 * (b["k"] - a["k"])
            dlo, dhi = den * lo, den * (hi - 1)
            if (num <= dlo) if tn else (num < dlo):
                if lo == 0 or moved > 0:  # pred true at lo, false at lo-1
                    return lo
                moved = -1
                j = lo - 1
                if a["lo"] == lo:
                    a = (self.make_piece(a["s"], a["e"] - 1, sm) if a["lo"] > self.cut[a["s"]]
                         else self.piece_at(s0, sm, j))
                if b["lo"] == lo:
                    b = (self.make_piece(b["s"], b["e"] - 1, s1) if b["lo"] > self.cut[b["s"]]
                         else self.piece_at(sm, s1, j))
            elif (num > dhi) if tn else (num >= dhi):
                if hi == W or moved < 0:  # pred false at hi-1, true at hi
                    return hi
                moved = 1
                j = hi
                if a["hi"] == hi:
                    seg_hi = self.cut[a["s"] + 1] if a["s"] + 1 < sm else W
                    a = self.make_piece(a["s"], a["e"] + 1, sm) if hi < seg_hi else self.piece_at(s0, sm, j)
                if b["hi"] == hi:
                    seg_hi = self.cut[b["s"] + 1] if b["s"] + 1 < s1 else W
                    b = self.make_piece(b["s"], b["e"] + 1, s1) if hi < seg_hi else self.piece_at(sm, s1, j)
            else:
                q = num // den
                return (q + (1 if num != q * den else 0)) if tn else q + 1
        raise RuntimeError("walk did not terminate")

    def cross_seg(self, s0, sm, s, max_steps=100000):
        """First column where segment s (full-domain stack, s >= sm) beats group
        A = [s0, sm) -- the lane-parallel merge: x_AB = min over s in B."""
        W, L, tn = self.W, self.L, self.tn
        st = self.stk[s]
        if not st:
            return W
        p0 = min(s * L, W - 1)

        def bpiece(e):
            k, start = st[e]
            return dict(e=e, k=k, g=self.g[k], lo=start, hi=st[e + 1][1] if e + 1 < len(st) else W)

        b = bpiece(self.entry(s, p0))
        a = self.piece_at(s0, sm, p0)
        if a is None:
            return 0
        moved = 0
        for _ in range(max_steps):
            lo, hi = max(a["lo"], b["lo"]), min(a["hi"], b["hi"])
            num = b["g"] - a["g"] + b["k"] ** 2 - a["k"] ** 2
            den = 2 * (b["k"] - a["k"])
            if (num <= den * lo) if tn else (num < den * lo):
                if lo == 0 or moved > 0:
                    return lo
                moved = -1
                if a["lo"] == lo:
                    a = (self.make_piece(a["s"], a["e"] - 1, sm) if a["lo"] > self.cut[a["s"]]
                         else self.piece_at(s0, sm, lo - 1))
                if b["lo"] == lo:
                    b = bpiece(b["e"] - 1)
            elif (num > den * (hi - 1)) if tn else (num >= den * (hi - 1)):
                if hi == W or moved < 0:
                    return hi
                moved = 1
                if a["hi"] == hi:
                    seg_hi = self.cut[a["s"] + 1] if a["s"] + 1 < sm else W
                    a = self.make_piece(a["s"], a["e"] + 1, sm) if hi < seg_hi else self.piece_at(s0, sm, hi)
                if b["hi"] == hi:
                    b = bpiece(b["e"] + 1)
            else:
                q = num // den
                return (q + (1 if num != q * den else 0)) if tn else q + 1
        raise RuntimeError("walk did not terminate")

    def E_group(self, s0, s1, j):
        p = self.piece_at(s0, s1, j)
        return None if p is None else p["g"] + (j - p["k"]) ** 2

    def beats(self, s0, sm, s1, j):
        eb, ea = self.E_group(sm, s1, j), self.E_group(s0, sm, j)
        if eb is None:
            return False
        if ea is None:
            return True
        return eb <= ea if self.tn else eb < ea

    def probe_merge(self, s0, sm, s1, P, stats=None):
        """P-ary probe search for the takeover column (mirrors k_rows.cu).
        Round 0 probes c-1 and c (c = B's first column: dense rows end here)
        and spreads the other P-2 probes uniformly; later rounds split the
        remaining bracket uniformly."""
        W, L = self.W, self.L
        lo, hi = 0, W            # x in [lo, hi]; pred(hi) true or hi == W
        c = min(sm * L, W - 1)
        rounds = 0
        while hi > lo:
            n = hi - lo
            if rounds == 0:
                ps = []
                for q in range(P):
                    if q < 2:
                        p = c - 1 + q
                    elif P >= 4 and q == 2:
                        p = 0
                    elif P >= 4 and q == P - 1:
                        p = W - 1
                    else:
                        p = lo + ((q - (2 if P >= 4 else 1)) * n) // (P - 3 if P >= 4 else P - 1)
                    ps.append(p)
                ps.sort()
            else:
                ps = [lo + ((q + 1) * n) // (P + 1) for q in range(P)]
            ps = [min(max(p, lo), hi - 1) for p in ps]
            rounds += 1
            bits = [self.beats(s0, sm, s1, p) for p in ps]
            f = next((q for q in range(P) if bits[q]), None)
            if f is None:
                lo = ps[-1] + 1
            else:
                hi = ps[f]
                if f > 0:
                    lo = ps[f - 1] + 1
        if stats is not None:
            stats.append(rounds)
        return lo

    def merge_all(self, lane_parallel=True):
        T = self.T
        G = 2
        while G <= T:
            half = G // 2
            if lane_parallel == "probe":
                P = min(G, 32)
                xs = {gb: self.probe_merge(gb, gb + half, gb + G, P, self.stats) for gb in range(0, T, G)}
            elif lane_parallel:
                xs = {gb: min(self.cross_seg(gb, gb + half, t) for t in range(gb + half, gb + G))
                      for gb in range(0, T, G)}
            else:
                xs = {gb: self.takeover(gb, gb + half, gb + G) for gb in range(0, T, G)}
            for s in range(T):
                gb = s & ~(G - 1)
                x = xs[gb]
                self.cut[s] = max(self.cut[s], x) if (s - gb) >= half else min(self.cut[s], x)
            G *= 2

    def fill(self):
        """(D, owner column) per j, None for an empty row."""
        out = []
        for j in range(self.W):
            s = self.owner(0, self.T, j)
            if not self.stk[s]:
                out.append((None, None))
                continue
            k = self.stk[s][self.entry(s, j)][0]
            out.append((self.g[k] + (j - k) ** 2, k))
        return out


def row_envelope(g, T, L, take_new=False, lane_parallel=True):
    r = Row(g, T, L, take_new)
    r.merge_all(lane_parallel)
    return r.fill()


def brute(g, take_new=False):
    W = len(g)
    out = []
    for j in range(W):
        best = None
        for k in range(W):
            if g[k] is None:
                continue
            d = g[k] + (j - k) ** 2
            if best is None or d < best[0] or (take_new and d == best[0]):
                best = (d, k)
        out.append(best if best else (None, None))
    return out
