// k_rows.cu -- stage 2 of the separable EDT: the per-row lower envelope of
// parabolas D_k(j) = g_k + (j-k)^2, g_k = (i - nearest_row_k)^2.
//
// Replaces envelope_rows / build_row_envelope / meijster_scan
// (exact_edt.cpp:190-283) and the label assembly of voronoi_labels
// (exact_edt.cpp:362-369).  The reference walks a row serially with one
// std::vector stack per row; here a row is owned by T threads (T*L >= cols,
// L = 2^k columns per thread, compile-time) of one CTA, in shared memory:
//
//  1. build   each thread runs the reference's stack algorithm (Meijster,
//             exact integer boundaries, exact_edt.cpp:200-223) over ITS L
//             columns: the lower envelope of its segment's parabolas over the
//             whole domain [0, cols), as a stack of (column, start) entries;
//  2. merge   log2(T) levels of pairwise merges of adjacent segment groups
//             A < B.  E_A - E_B is strictly increasing in j (all columns of A
//             are left of B's), so B takes over from A at ONE column x; every
//             segment keeps a "cut", the first column it may own inside its
//             current group.  The P = min(G, 32) lanes of a merge find x by a
//             P-ary probe search: each round evaluates "B beats A" at P
//             columns of the bracket [lo, hi] (the group envelope at a column
//             is a binary search over cuts, then over that segment's stack).
//             The bracket starts at (zl(A), zf(B)] -- A's last and B's first
//             column with an object pixel on this row own themselves -- so on
//             dense rows most merges need no probe; round 0 also probes c-1, c
//             (c = B's first column) and both row ends.  Rows with at most
//             kCompact candidates left skip the tree: one lane re-runs the
//             stack algorithm over all segment stacks.
//  3. fill    each thread walks its own columns along cuts and stacks (the
//             owner column is monotone in j) and writes D, sqrt(D), the
//             label and/or the nearest column.
//
// Tie rules are order-independent and therefore exact under any merge order:
// keep_old (the label rule, exact_edt.cpp:205/:363) hands a tie to the
// SMALLER column everywhere -- in the stacks (floor(x)+1 boundaries) and in
// the merges (B takes over only where strictly smaller); take_new
// (meijster_scan's nearest_col, exact_edt.cpp:275) to the LARGER column.
// The label of a cell is (nearest_row_k, k) of its owner k; stage 1 already
// resolved vertical ties to the upper feature.
//
// All arithmetic is exact 32/64-bit integer: every value is bounded by
// (rows-1)^2 + (cols-1)^2 <= 2^31-2 (DFC_MAX_SQDIST, SURVEY.md finding 7).
#include "dfc_kernels.cuh"

namespace dfc {

// Rows whose segment stacks hold at most this many candidates in total are
// merged by one lane instead of the merge tree (C3-like sparse rows).
constexpr int kCompact = 64;

template <int L>
struct RowLayout {
    static constexpr int kLog = L == 4 ? 2 : L == 8 ? 3 : L == 16 ? 4 : L == 32 ? 5 : L == 64 ? 6 : 7;
    // Segment-padded index of column j in the per-row nr array: each thread's
    // L columns are followed by 2 pad halfwords so the build phase (thread t
    // reads column t*L + x) is bank-conflict free (word stride L/2+1 is odd).
    __device__ static __forceinline__ int nidx(int j) { return (j >> kLog) * (L + 2) + (j & (L - 1)); }
    static constexpr int stk_stride = L + 1;  // odd word stride: conflict-free
};

template <int L, bool TAKE_NEW>
struct RowCtx {
    const uint16_t* nrs;
    const uint32_t* stk;
    const int* cut;
    const int* cnt;
    uint32_t i;
    int W;

    __device__ __forceinline__ uint32_t g_of(int k) const {
        const uint32_t r = nrs[RowLayout<L>::nidx(k)];
        const uint32_t a = i > r ? i - r : r - i;
        return a * a;
    }
    __device__ __forceinline__ int start(int s, int e) const {
        return (int)(stk[s * RowLayout<L>::stk_stride + e] >> 16);
    }
    // last s in [s0, s1) with cut[s] <= j (cut[s0] == 0 inside a group)
    __device__ __forceinline__ int owner(int s0, int s1, int j) const {
        int lo = s0, hi = s1 - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cut[mid] <= j) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
    // last entry of segment s with start <= j (start(s, 0) == 0)
    __device__ __forceinline__ int entry(int s, int n, int j) const {
        const uint32_t* st = stk + s * RowLayout<L>::stk_stride;
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int)(st[mid] >> 16) <= j) lo = mid; else hi = mid - 1;
        }
        return lo;
    }
    // Envelope of group [s0, s1) at column j (kInfU if the group is empty).
    __device__ __forceinline__ uint32_t env(int s0, int s1, int j) const {
        const int s = owner(s0, s1, j);
        const int n = cnt[s];
        if (n == 0) return kInfU;
        const uint32_t ent = stk[s * RowLayout<L>::stk_stride + entry(s, n, j)];
        const int k = (int)(ent & 0xffffu);
        return g_of(k) + (uint32_t)((j - k) * (j - k));
    }
    // Does group B = [sm, s1) beat group A = [s0, sm) at column j?  Monotone
    // in j (false ... false true ... true), E_A - E_B strictly increasing.
    __device__ __forceinline__ bool beats(int s0, int sm, int s1, int j) const {
        const uint32_t eb = env(sm, s1, j), ea = env(s0, sm, j);
        return TAKE_NEW ? (eb <= ea && eb != kInfU) : (eb < ea);
    }
};

template <int L, bool TAKE_NEW>
__device__ __forceinline__ void rows_group(const RowArgs& a, int64_t grp);

template <int L, bool TAKE_NEW>
__global__ void __launch_bounds__(1024) k_rows(RowArgs a) {
    if (a.row_list == nullptr) {
        rows_group<L, TAKE_NEW>(a, blockIdx.x);
        return;
    }
    // fallback mode (rows the streaming kernel could not hold): grid-stride
    // over the listed rows; the trip count is uniform per CTA
    const int64_t n = *a.row_count;
    for (int64_t grp = blockIdx.x; grp * a.R < n; grp += gridDim.x) {
        rows_group<L, TAKE_NEW>(a, grp);
        __syncthreads();
    }
}

template <int L, bool TAKE_NEW>
__device__ __forceinline__ void rows_group(const RowArgs& a, int64_t grp) {
    using LY = RowLayout<L>;
    extern __shared__ uint32_t smem[];
    const int T = a.T;
    const int rho = threadIdx.x / T;          // row within the CTA
    const int s = threadIdx.x - rho * T;      // segment (thread) within the row
    int64_t row = grp * a.R + rho;
    bool active = row < a.total_rows;
    if (a.row_list) {
        active = row < *a.row_count;
        row = active ? a.row_list[row] : 0;
    }
    if (a.row_done) {  // rows k_rows_dense / k_rows_lr already wrote
        if (active) {
            const uint8_t rd = a.row_done[row];
            const int pl = (int)(row / a.H);
            if (rd == 1 || pts_plane(a.plane_counts, pl, a.pts_gate) ||
                (a.lr_gate && rd != 2 && lr_plane(a.plane_counts, pl, a.H, a.W)))
                active = false;
        }
        if (__syncthreads_and(!active)) return;  // CTA-uniform
    }
    const int img = active ? (int)(row / a.H) : 0;
    const uint32_t i = active ? (uint32_t)(row - (int64_t)img * a.H) : 0u;
    const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;  // g = (gi - nr)^2, global row
    const int W = a.W;

    // sparse plane (fewer object pixels than columns, e.g. C3): candidate
    // columns are few, so the build visits them through per-segment bit masks
    const bool sparse = L == 32 && active && a.plane_counts && a.tile_cols >= W &&
                        a.plane_counts[img] < (unsigned long long)W;
    uint32_t* base = smem + rho * a.row_smem_words;
    uint16_t* nrs = reinterpret_cast<uint16_t*>(base);            // [T*(L+2)]
    uint32_t* stk = base + (T * (L + 2)) / 2;                     // [T*(L+1)]
    int* cut = reinterpret_cast<int*>(stk + T * LY::stk_stride);  // [T]
    int* cnt = cut + T;                                           // [T]
    int* xs = cnt + T;                                            // [T/32] per warp: takeover / census
    int* nzw = xs + (T >> 5);                                     // [T/32] warp has candidates
    uint32_t* cmp = reinterpret_cast<uint32_t*>(nzw + (T >> 5));  // [kCompact+2] compact envelope
    int* wzf = reinterpret_cast<int*>(cmp + kCompact + 2);        // [T/32] first zero column of a warp's group
    int* wzl = wzf + (T >> 5);                                    // [T/32] last zero column of a warp's group

    // ---- 0. stage the row's nearest-row values (coalesced 4-byte loads) ----
    if (active) {
        const uint16_t* rowp = a.nr + img * a.nr_img_stride + (int64_t)i * a.Wp;
        const int npairs = (W + 1) >> 1;
        if (sparse) {
            // one tile, 32-column segments: the warp's 32 pairs are 2 segments;
            // their candidate masks (bit x: column c0+x has an object in its
            // column) come from two ballots, parked in cut[] until the build
            const uint32_t* src = reinterpret_cast<const uint32_t*>(rowp);
            const int lane = threadIdx.x & 31;
            for (int q0 = s - lane; q0 < npairs; q0 += T) {
                const int q = q0 + lane;
                uint32_t v = 0xffffffffu;
                if (q < npairs) {
                    v = __ldg(src + q);
                    *reinterpret_cast<uint32_t*>(nrs + LY::nidx(2 * q)) = v;
                }
                const uint32_t b0 = __ballot_sync(0xffffffffu, (v & 0xffffu) != kNoRow && 2 * q < W);
                const uint32_t b1 = __ballot_sync(0xffffffffu, (v >> 16) != kNoRow && 2 * q + 1 < W);
                if ((lane & 15) == 0) {  // lanes 0 / 16: segment (2 q0 + 2 lane) / 32
                    uint32_t e0 = (b0 >> lane) & 0xffffu, e1 = (b1 >> lane) & 0xffffu;
                    // spread 16 bits to the even positions (pairs -> columns)
                    e0 = (e0 | (e0 << 8)) & 0x00ff00ffu;  e1 = (e1 | (e1 << 8)) & 0x00ff00ffu;
                    e0 = (e0 | (e0 << 4)) & 0x0f0f0f0fu;  e1 = (e1 | (e1 << 4)) & 0x0f0f0f0fu;
                    e0 = (e0 | (e0 << 2)) & 0x33333333u;  e1 = (e1 | (e1 << 2)) & 0x33333333u;
                    e0 = (e0 | (e0 << 1)) & 0x55555555u;  e1 = (e1 | (e1 << 1)) & 0x55555555u;
                    const int sg = (2 * q0 + 2 * lane) >> 5;
                    if (sg < T) cut[sg] = (int)(e0 | (e1 << 1));
                }
            }
        } else if (a.tile_cols >= W) {  // one tile: the row is contiguous
            const uint32_t* src = reinterpret_cast<const uint32_t*>(rowp);
            for (int q = s; q < npairs; q += T)
                *reinterpret_cast<uint32_t*>(nrs + LY::nidx(2 * q)) = __ldg(src + q);
        } else {                 // row striped over column tiles (received all-to-all blocks)
            int t = (2 * s) / a.tile_cols;  // tile of column 2q, advanced incrementally
            for (int q = s; q < npairs; q += T) {
                const int j = 2 * q;
                while (j >= (t + 1) * a.tile_cols) ++t;
                const uint16_t* p = rowp + t * a.tile_stride + (j - t * a.tile_cols);
                *reinterpret_cast<uint32_t*>(nrs + LY::nidx(j)) = __ldg(reinterpret_cast<const uint32_t*>(p));
            }
        }
    }
    __syncthreads();

    // ---- 1. per-segment envelope (exact_edt.cpp:208-223) ----
    int zf = W, zl = -1;  // first / last column with an object pixel ON this row (g = 0)
    {
        const int c0 = s * L, c1 = min(c0 + L, W);
        uint32_t* st = stk + s * LY::stk_stride;
        int n = 0;
        int tk = 0, ts = 0;   // top entry: column, start
        int tg = 0;           // top entry: vertical value
        if (active) {
            // One event per iteration -- pop the top, or consume column m
            // (push or skip) -- instead of a nested pop loop: lanes of a warp
            // reconverge every iteration.  On sparse planes only the candidate
            // columns are visited (bit mask from the staging).
            const uint16_t* seg_nr = nrs + s * (L + 2);
            uint32_t rem = sparse ? (uint32_t)cut[s] : 0u;
            const bool by_mask = sparse;
            int m = c0;
            int gm = -1;  // vertical value of column m, -1 = no feature (:212)
            auto load_m = [&]() {
                if (by_mask) {
                    if (rem) {
                        const int x = __ffs(rem) - 1;
                        rem &= rem - 1;
                        m = c0 + x;
                        const uint32_t r = seg_nr[x];
                        const int am = (int)(gi > r ? gi - r : r - gi);
                        gm = am * am;
                    } else {
                        m = c1;
                    }
                    return;
                }
                const uint32_t r = m < c1 ? nrs[LY::nidx(m)] : kNoRow;
                const int am = (int)(gi > r ? gi - r : r - gi);
                gm = r == kNoRow ? -1 : am * am;
            };
            if (by_mask) load_m();
            else {
                const uint32_t r = m < c1 ? nrs[LY::nidx(m)] : kNoRow;
                const int am = (int)(gi > r ? gi - r : r - gi);
                gm = r == kNoRow ? -1 : am * am;
            }
            while (m < c1) {
                if (gm == 0) {
                    zf = min(zf, m);
                    zl = m;
                }
                if (gm == 0 && n > 0 && tg == 0 && tk == m - 1) {
                    // run of object pixels: the new zero parabola starts exactly at m
                    // and pops nothing (num = 2m-1 > 2*ts, start = m, push since m < W)
                    st[n++] = (uint32_t)m | ((uint32_t)m << 16);
                    tk = m;
                    ts = m;
                    if (!by_mask) ++m;
                    load_m();
                    continue;
                }
                bool consume = true;
                int num = 0;
                uint32_t den = 1;
                if (gm >= 0 && n > 0) {
                    // num = v_m - v_k - k^2 + m^2 fits int32 (|.| < 2^31); ts*den < 2^32
                    num = gm - tg + (m * m - tk * tk);
                    den = 2u * (uint32_t)(m - tk);
                    const uint32_t lim = (uint32_t)ts * den;  // start <= js[idx]  (:214)
                    if (num < 0 || (TAKE_NEW ? (uint32_t)num <= lim : (uint32_t)num < lim)) {
                        consume = false;  // pop
                        if (--n > 0) {
                            const uint32_t e = st[n - 1];
                            tk = (int)(e & 0xffffu);
                            ts = (int)(e >> 16);
                            const uint32_t rk = nrs[LY::nidx(tk)];
                            const int ak = (int)(gi > rk ? gi - rk : rk - gi);
                            tg = ak * ak;
                        }
                    }
                }
                if (consume) {
                    if (gm >= 0) {
                        int start = 0;
                        bool push = true;
                        if (n > 0) {
                            // push iff start <= cols-1 (:218); here 0 <= num
                            const uint32_t lim = (uint32_t)(W - 1) * den;
                            push = TAKE_NEW ? (uint32_t)num <= lim : (uint32_t)num < lim;
                            const uint32_t q = small_udiv((uint32_t)num, den);
                            // keep_old: floor(x)+1 ; take_new: ceil(x)   (:205)
                            start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * den)) : (int)q + 1;
                        }
                        if (push) {
                            st[n++] = (uint32_t)m | ((uint32_t)start << 16);
                            tk = m;
                            ts = start;
                            tg = gm;
                        }
                    }
                    if (!by_mask) ++m;
                    load_m();
                }
            }
        }
        cnt[s] = n;
        cut[s] = 0;
    }
    __syncthreads();

    RowCtx<L, TAKE_NEW> cx{nrs, stk, cut, cnt, gi, W};

    // ---- 1b. row census: candidates per row, which warps have any ----
    const int lane = threadIdx.x & 31;
    const int my_cnt = active ? cnt[s] : 0;
    const uint32_t nzmask = __ballot_sync(0xffffffffu, my_cnt > 0);
    int tot = my_cnt;
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (T > 32) {
        if (lane == 0) {
            xs[s >> 5] = tot;
            nzw[s >> 5] = nzmask != 0;
        }
        __syncthreads();
        tot = 0;
        for (int w = 0; w < (T >> 5); ++w) tot += xs[w];
    }

    // (CTA-uniform choice: rows sharing a CTA must run the same barriers)
    if (__syncthreads_and(tot <= kCompact)) {
        // ---- 2'. sparse row: one lane runs the reference stack algorithm
        // (exact_edt.cpp:208-223) over the surviving candidates of all
        // segments, in column order; the result becomes a single segment.
        if (s == 0 && active) {
            int n = 0, tk = 0, ts = 0, tg = 0;
            for (int sg = 0; sg < T; ++sg) {
                const int cn = cnt[sg];
                for (int e = 0; e < cn; ++e) {
                    const int m = (int)(stk[sg * LY::stk_stride + e] & 0xffffu);
                    const int gm = (int)cx.g_of(m);
                    int start = 0;
                    bool push = true;
                    while (n > 0) {
                        const int num = gm - tg + (m * m - tk * tk);
                        const uint32_t den = 2u * (uint32_t)(m - tk);
                        const uint32_t lim = (uint32_t)ts * den;
                        if (num < 0 || (TAKE_NEW ? (uint32_t)num <= lim : (uint32_t)num < lim)) {
                            if (--n > 0) {
                                const uint32_t ent = cmp[n - 1];
                                tk = (int)(ent & 0xffffu);
                                ts = (int)(ent >> 16);
                                tg = (int)cx.g_of(tk);
                            }
                            continue;
                        }
                        const uint32_t lim2 = (uint32_t)(W - 1) * den;
                        push = TAKE_NEW ? (uint32_t)num <= lim2 : (uint32_t)num < lim2;
                        const uint32_t qd = small_udiv((uint32_t)num, den);
                        start = TAKE_NEW ? (int)(qd + ((uint32_t)num != qd * den)) : (int)qd + 1;
                        break;
                    }
                    if (push) {
                        cmp[n++] = (uint32_t)m | ((uint32_t)start << 16);
                        tk = m;
                        ts = start;
                        tg = gm;
                    }
                }
            }
            for (int e = 0; e < n; ++e) stk[e] = cmp[e];  // all segment stacks already consumed
            cnt[0] = n;
        }
        if (T > 32) __syncthreads(); else __syncwarp();
        if (active && s > 0) cut[s] = W;   // segment 0 owns the whole row
        __syncthreads();
    } else {
    // ---- 2. merge adjacent segment groups: P-ary probe search ----
    // The P = min(G, 32) lanes of a merge evaluate "B beats A" at P columns
    // per round.  Round 0 probes c-1 and c (c = B's first column, where dense
    // rows take over) and spreads the rest over the row; later rounds split
    // the remaining bracket [lo, hi] uniformly.  The outcome is reduced
    // order-independently: hi = min column where B beats, lo = 1 + max column
    // where it does not.  G <= 32: groups live inside a warp and search in
    // lockstep; G > 32: the group's first warp searches, the others wait.
    for (int G = 2; G <= T; G <<= 1) {
        const int gb = s & ~(G - 1);
        const int half = G >> 1;
        const int P = G < 32 ? G : 32;
        const int q = s - gb;
        if (G > 32) __syncthreads();  // every warp's cuts of the previous level
        // zero columns of both halves: zf/zl hold my (G/2)-group's first/last
        int zfA, zlA, zfB, zlB;
        if (G <= 32) {  // (rows narrower than a warp share it: lane - s is the row's first lane)
            const int la = (lane - s + gb) & 31, lb = (lane - s + gb + half) & 31;
            zfA = __shfl_sync(0xffffffffu, zf, la);
            zlA = __shfl_sync(0xffffffffu, zl, la);
            zfB = __shfl_sync(0xffffffffu, zf, lb);
            zlB = __shfl_sync(0xffffffffu, zl, lb);
        } else {
            zfA = wzf[gb >> 5];
            zlA = wzl[gb >> 5];
            zfB = wzf[(gb + half) >> 5];
            zlB = wzl[(gb + half) >> 5];
        }
        if (q < 32) {                 // warp-uniform: whole warps probe or not
            const int c = min((gb + half) * L, W - 1);
            const float rP1 = 1.0f / (float)(P + 1);
            const float rPm1 = P >= 4 ? 1.0f / (float)(P - 3) : P > 2 ? 1.0f / (float)(P - 1) : 0.f;
            int lo = 0, hi = W;
            // a side without any finite parabola decides the merge at once
            bool hasA, hasB;
            if (G <= 32) {
                const uint32_t hm = half == 32 ? 0xffffffffu : ((1u << half) - 1u);
                hasA = ((nzmask >> (gb & 31)) & hm) != 0;
                hasB = ((nzmask >> ((gb & 31) + half)) & hm) != 0;
            } else {
                hasA = hasB = false;
                for (int w = gb >> 5; w < (gb + half) >> 5; ++w) hasA |= nzw[w] != 0;
                for (int w = (gb + half) >> 5; w < (gb + G) >> 5; ++w) hasB |= nzw[w] != 0;
            }
            if (!hasB) lo = hi = W;
            else if (!hasA) lo = hi = 0;
            else {
                // A owns its last zero column zl(A) (D = 0, unique), B its first
                // zf(B): B takes over inside (zl(A), zf(B)] -- on dense rows an
                // empty bracket, no probe round at all.
                if (zlA >= 0) lo = zlA + 1;
                if (zfB < W) hi = zfB;
            }
            bool first = true;
            while (__any_sync(0xffffffffu, active && hi > lo)) {
                const int n = hi - lo;
                int p;
                if (first) {
                    // c-1, c (dense rows take over at B's first column), both ends
                    // (sparse rows: one side often owns everything), uniform rest
                    if (q < 2) p = c - 1 + q;
                    else if (P >= 4 && q == 2) p = 0;
                    else if (P >= 4 && q == P - 1) p = W - 1;
                    else p = lo + __float2int_rz((float)((q - (P >= 4 ? 2 : 1)) * n) * rPm1);
                }
                else p = lo + __float2int_rz((float)((q + 1) * n) * rP1);
                p = min(max(p, lo), hi - 1);
                const bool live = active && hi > lo;
                const bool bt = live && cx.beats(gb, gb + half, gb + G, p);
                int t = live && bt ? p : W;             // first column where B beats
                int f = live && !bt ? p : -1;           // last column where it does not
                for (int o = 1; o < P; o <<= 1) {
                    t = min(t, __shfl_xor_sync(0xffffffffu, t, o));
                    f = max(f, __shfl_xor_sync(0xffffffffu, f, o));
                }
                if (live) {
                    hi = min(hi, t);
                    lo = max(lo, f + 1);
                }
                first = false;
            }
            if (G > 32 && q == 0) xs[gb >> 5] = lo;
            if (G <= 32 && active) cut[s] = q >= half ? max(cut[s], lo) : min(cut[s], lo);
        }
        if (G > 32) {
            __syncthreads();
            if (active) cut[s] = q >= half ? max(cut[s], xs[gb >> 5]) : min(cut[s], xs[gb >> 5]);
        }
        zf = min(zfA, zfB);  // the merged group's zero columns
        zl = max(zlA, zlB);
        if (G >= 32 && lane == 0) {  // read at the next level after its barrier
            wzf[s >> 5] = zf;
            wzl[s >> 5] = zl;
        }
        __syncwarp();
    }
    __syncthreads();
    }  // dense row

    // ---- 3. fill this thread's columns ----
    if (!active) return;
    const int c0 = s * L, c1 = min(c0 + L, W);
    if (c0 >= W) return;
    int sg = cx.owner(0, T, c0);
    int seg_end = sg + 1 < T ? cut[sg + 1] : W;
    int n = cnt[sg];
    int e = n > 0 ? cx.entry(sg, n, c0) : 0;
    uint32_t k = 0, rr = kNoRow, gk = kInfU;
    int next_start = W;
    auto load_entry = [&]() {
        if (n == 0) { k = 0; rr = kNoRow; gk = kInfU; next_start = W; return; }
        const uint32_t ent = stk[sg * LY::stk_stride + e];
        k = ent & 0xffffu;
        rr = nrs[LY::nidx((int)k)];
        const uint32_t av = gi > rr ? gi - rr : rr - gi;
        gk = av * av;
        next_start = e + 1 < n ? (int)(stk[sg * LY::stk_stride + e + 1] >> 16) : W;
    };
    load_entry();

    int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + img * a.sD) + (int64_t)i * W : nullptr;
    float* Srow = a.S ? reinterpret_cast<float*>(a.S + img * a.sS) + (int64_t)i * W : nullptr;
    int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + img * a.sL) + (int64_t)i * W : nullptr;
    int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + img * a.sN) + (int64_t)i * W : nullptr;

    auto cell = [&](int j, int32_t& d, uint32_t& kk, uint32_t& rk) {
        if (j >= seg_end) {
            while (sg + 1 < T && cut[sg + 1] <= j) ++sg;
            seg_end = sg + 1 < T ? cut[sg + 1] : W;
            n = cnt[sg];
            e = n > 0 ? cx.entry(sg, n, j) : 0;
            load_entry();
        }
        while (j >= next_start) {
            ++e;
            load_entry();
        }
        kk = k;
        rk = rr;
        if (gk == kInfU) {
            d = DFC_INF_I32;
        } else {
            const int dj = j - (int)k;
            d = (int32_t)(gk + (uint32_t)(dj * dj));
        }
    };
    auto lab_of = [&](int32_t d, uint32_t kk, uint32_t rk) -> int32_t {
        return d == DFC_INF_I32 ? -1 : (int32_t)(rk * (uint32_t)W + kk);
    };
    auto col_of = [&](int32_t d, uint32_t kk) -> int32_t { return d == DFC_INF_I32 ? -1 : (int32_t)kk; };

    if (a.vec) {
        for (int j = c0; j < c1; j += 4) {
            int4 d4;
            uint32_t k0, k1, k2, k3, r0, r1, r2, r3;
            cell(j + 0, d4.x, k0, r0);
            cell(j + 1, d4.y, k1, r1);
            cell(j + 2, d4.z, k2, r2);
            cell(j + 3, d4.w, k3, r3);
            if (Drow) __stcs(reinterpret_cast<int4*>(Drow + j), d4);
            if (Srow) {
                const float4 f4 = make_float4(dist_f32(d4.x), dist_f32(d4.y), dist_f32(d4.z),
                                              dist_f32(d4.w));
                __stcs(reinterpret_cast<float4*>(Srow + j), f4);
            }
            if (Lrow)
                __stcs(reinterpret_cast<int4*>(Lrow + j), make_int4(lab_of(d4.x, k0, r0), lab_of(d4.y, k1, r1),
                                                                   lab_of(d4.z, k2, r2), lab_of(d4.w, k3, r3)));
            if (Nrow)
                __stcs(reinterpret_cast<int4*>(Nrow + j),
                       make_int4(col_of(d4.x, k0), col_of(d4.y, k1), col_of(d4.z, k2), col_of(d4.w, k3)));
        }
    } else {
        for (int j = c0; j < c1; ++j) {
            int32_t d;
            uint32_t kk, rk;
            cell(j, d, kk, rk);
            if (Drow) Drow[j] = d;
            if (Srow) Srow[j] = dist_f32((uint32_t)d);
            if (Lrow) Lrow[j] = lab_of(d, kk, rk);
            if (Nrow) Nrow[j] = col_of(d, kk);
        }
    }
}

// Row-pass words of shared memory per row for a given (T, L).
inline int row_words(int T, int L) {
    return (T * (L + 2)) / 2 + T * (L + 1) + 2 * T + 4 * (T >> 5) + kCompact + 2;  // nrs, stacks, cut, cnt, ...
}

// Host-side dispatch over the compile-time segment length.
template <bool TAKE_NEW>
inline const void* rows_kernel_ptr(int L) {
    switch (L) {
        case 4: return (const void*)k_rows<4, TAKE_NEW>;
        case 8: return (const void*)k_rows<8, TAKE_NEW>;
        case 16: return (const void*)k_rows<16, TAKE_NEW>;
        case 32: return (const void*)k_rows<32, TAKE_NEW>;
        case 64: return (const void*)k_rows<64, TAKE_NEW>;
        default: return (const void*)k_rows<128, TAKE_NEW>;
    }
}

}  // namespace dfc
