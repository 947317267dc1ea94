// k_rows.cu -- stage 2 of the separable EDT: the per-row lower envelope of
// parabolas D_k(j) = g_k + (j-k)^2, g_k = (i - nearest_row_k)^2.
//
// Replaces envelope_rows / build_row_envelope / meijster_scan
// (exact_edt.cpp:190-283) and the label assembly of voronoi_labels
// (exact_edt.cpp:362-369).  The reference walks a row serially with one
// std::vector stack per row; here a row is owned by T threads (T*L >= cols,
// L columns per thread) of one CTA and processed in three phases, all in
// shared memory:
//
//  1. build   each thread runs the reference's stack algorithm (Meijster,
//             exact integer boundaries, exact_edt.cpp:200-223) over ITS L
//             columns, producing the lower envelope of its segment's
//             parabolas over the whole domain [0, cols);
//  2. merge   log2(T) levels of pairwise merges of adjacent segment groups.
//             For groups A < B (all columns of A left of B) E_A - E_B is
//             strictly increasing in j, so B takes over from A at ONE column
//             x (the first j where B beats A under the tie rule).  The
//             2^(l+1) threads of a merge find x with a (2^(l+1)+1)-ary search,
//             evaluating both group envelopes at their probe columns.  Each
//             segment keeps a "cut": the first column it may own.
//  3. fill    each thread walks its own columns, following cuts and segment
//             stacks (owners are monotone in j), and writes D, sqrt(D),
//             label and/or nearest column.
//
// Tie rules are order-independent and therefore exact under any merge order:
// keep_old (the label rule, exact_edt.cpp:205/:363) hands a tie to the
// SMALLER column everywhere -- in the segment stacks (floor(x)+1 boundaries)
// and in the merges ("B beats A" only when strictly smaller); take_new
// (meijster_scan's nearest_col, exact_edt.cpp:275) to the LARGER column.
// The label of a cell is then (nearest_row_k, k) of its owner k, the upper
// feature on vertical ties (stage 1).
//
// All arithmetic is int32/int64 and exact: every value is bounded by
// (rows-1)^2 + (cols-1)^2 <= 2^31-2 (DFC_MAX_SQDIST), see SURVEY.md finding 7.
#include "dfc_kernels.cuh"

namespace dfc {


// Segment-padded index of column j in the per-row nr array: each thread's L
// columns are followed by 2 pad halfwords so the build phase (thread t reads
// column t*L + x) is bank-conflict free (word stride L/2+1 is odd).
__device__ __forceinline__ int nidx(int j, int L) { return (j / L) * (L + 2) + (j % L); }

struct RowSmem {
    uint16_t* nrs;   // [T*(L+2)]
    uint32_t* stk;   // [T*(L+1)]  entry = k | start << 16
    int* cut;        // [T]
    int* cnt;        // [T]
};

__device__ __forceinline__ RowSmem row_smem(uint32_t* base, int T, int L) {
    RowSmem s;
    s.nrs = reinterpret_cast<uint16_t*>(base);
    uint32_t* p = base + (T * (L + 2)) / 2;
    s.stk = p;
    p += T * (L + 1);
    s.cut = reinterpret_cast<int*>(p);
    p += T;
    s.cnt = reinterpret_cast<int*>(p);
    return s;
}

__device__ __forceinline__ uint32_t g_of(const RowSmem& sm, int L, uint32_t i, uint32_t k) {
    const uint32_t r = sm.nrs[nidx((int)k, L)];
    const uint32_t a = i > r ? i - r : r - i;
    return a * a;
}

// Envelope value of one segment's stack at column j (kInfU if the segment has
// no finite parabola); also returns the serving entry.
__device__ __forceinline__ uint32_t eval_seg(const RowSmem& sm, int L, uint32_t i, int s, int j) {
    const int n = sm.cnt[s];
    if (n == 0) return kInfU;
    const uint32_t* st = sm.stk + s * (L + 1);
    int lo = 0, hi = n - 1;  // last e with start(e) <= j; start(0) == 0
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((int)(st[mid] >> 16) <= j) lo = mid; else hi = mid - 1;
    }
    const uint32_t k = st[lo] & 0xffffu;
    const int dj = j - (int)k;
    return g_of(sm, L, i, k) + (uint32_t)(dj * dj);
}

// Owner segment of column j inside segments [s0, s1): the last s with cut[s] <= j.
__device__ __forceinline__ int owner_seg(const RowSmem& sm, int s0, int s1, int j) {
    int lo = s0, hi = s1 - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sm.cut[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <bool TAKE_NEW>
__device__ __forceinline__ bool beats(uint32_t eb, uint32_t ea) {
    return TAKE_NEW ? (eb <= ea && eb != kInfU) : (eb < ea);
}

template <bool TAKE_NEW>
__global__ void __launch_bounds__(1024) k_rows(RowArgs a) {
    extern __shared__ uint32_t smem[];
    const int T = a.T, L = a.L;
    const int rho = threadIdx.x / T;          // row within the CTA
    const int s = threadIdx.x - rho * T;      // segment (thread) within the row
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * a.R + rho;
    const bool active = row < a.total_rows;
    const int img = active ? (int)(row / a.H) : 0;
    const uint32_t i = active ? (uint32_t)(row - (int64_t)img * a.H) : 0u;
    const int W = a.W;
    RowSmem sm = row_smem(smem + rho * a.row_smem_words, T, L);

    // ---- 0. stage the row's nearest-row values (coalesced 4-byte loads) ----
    if (active) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a.nr + img * a.nr_img_stride +
                                                                (int64_t)i * a.Wp);
        const int npairs = (W + 1) >> 1;
        for (int q = s; q < npairs; q += T)
            *reinterpret_cast<uint32_t*>(sm.nrs + nidx(2 * q, L)) = __ldg(src + q);
    }
    __syncthreads();

    // ---- 1. per-segment envelope (exact_edt.cpp:208-223) ----
    {
        const int c0 = s * L, c1 = min(c0 + L, W);
        uint32_t* st = sm.stk + s * (L + 1);
        int n = 0;
        int tk = 0, ts = 0;   // top entry: column, start
        uint32_t tg = 0;      // top entry: vertical value
        if (active) {
            for (int m = c0; m < c1; ++m) {
                const uint32_t r = sm.nrs[nidx(m, L)];
                if (r == kNoRow) continue;  // sentinel vertex never enters (:212)
                const uint32_t am = i > r ? i - r : r - i;
                const uint32_t gm = am * am;
                int64_t num = 0, den = 1;
                while (n > 0) {
                    num = (int64_t)gm - (int64_t)tg + (int64_t)m * m - (int64_t)tk * tk;
                    den = 2 * (int64_t)(m - tk);
                    const int64_t lim = (int64_t)ts * den;  // start <= js[idx]  (:214)
                    if (TAKE_NEW ? (num <= lim) : (num < lim)) {
                        if (--n > 0) {
                            const uint32_t e = st[n - 1];
                            tk = (int)(e & 0xffffu);
                            ts = (int)(e >> 16);
                            tg = g_of(sm, L, i, (uint32_t)tk);
                        }
                    } else {
                        break;
                    }
                }
                int start = 0;
                if (n > 0) {
                    // push iff start <= cols-1 (:218); num >= 0 here
                    const int64_t lim = (int64_t)(W - 1) * den;
                    if (TAKE_NEW ? (num > lim) : (num >= lim)) continue;
                    const uint32_t q = small_udiv((uint32_t)num, (uint32_t)den);
                    // keep_old: floor(x)+1 ; take_new: ceil(x)   (:205)
                    start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * (uint32_t)den)) : (int)q + 1;
                }
                st[n++] = (uint32_t)m | ((uint32_t)start << 16);
                tk = m;
                ts = start;
                tg = gm;
            }
        }
        sm.cnt[s] = n;
        sm.cut[s] = 0;
    }
    __syncthreads();

    // ---- 2. merge adjacent segment groups ----
    for (int G = 2; G <= T; G <<= 1) {
        const int half = G >> 1;
        const int gb = (s / G) * G;
        const int q = s - gb;               // probe index within the merge
        const bool inB = q >= half;
        int lo = 0, hi = W;                 // takeover column x lies in [lo, hi]
        if (G <= 32) {
            const int sh = (threadIdx.x & 31) & ~(G - 1);
            const uint32_t gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
            while (__any_sync(0xffffffffu, active && hi > lo)) {
                const int n = hi - lo;
                const int p = lo + (n * (q + 1)) / (G + 1);
                bool bt = false;
                if (active && hi > lo) {
                    const int sa = owner_seg(sm, gb, gb + half, p);
                    const int sb = owner_seg(sm, gb + half, gb + G, p);
                    bt = beats<TAKE_NEW>(eval_seg(sm, L, i, sb, p), eval_seg(sm, L, i, sa, p));
                }
                const uint32_t bits = (__ballot_sync(0xffffffffu, bt) >> sh) & gmask;
                if (hi > lo) {
                    if (bits) {
                        const int qs = __ffs(bits) - 1;
                        const int nlo = qs > 0 ? lo + (n * qs) / (G + 1) + 1 : lo;
                        hi = lo + (n * (qs + 1)) / (G + 1);
                        lo = nlo;
                    } else {
                        lo = lo + (n * G) / (G + 1) + 1;
                    }
                }
            }
        } else {
            const int nw = G >> 5;              // warps per merge
            const int w0 = (rho * T + gb) >> 5; // first warp word of this merge
            for (;;) {
                const bool live = active && hi > lo;
                const int n = hi - lo;
                const int p = lo + (int)(((int64_t)n * (q + 1)) / (G + 1));
                bool bt = false;
                if (live) {
                    const int sa = owner_seg(sm, gb, gb + half, p);
                    const int sb = owner_seg(sm, gb + half, gb + G, p);
                    bt = beats<TAKE_NEW>(eval_seg(sm, L, i, sb, p), eval_seg(sm, L, i, sa, p));
                }
                const uint32_t w = __ballot_sync(0xffffffffu, bt);
                uint32_t* bal = reinterpret_cast<uint32_t*>(smem + a.R * a.row_smem_words);
                if (lane == 0) bal[threadIdx.x >> 5] = w;
                __syncthreads();
                if (live) {
                    int qs = -1;
                    for (int t = 0; t < nw; ++t) {
                        const uint32_t bw = bal[w0 + t];
                        if (bw) { qs = 32 * t + __ffs(bw) - 1; break; }
                    }
                    if (qs >= 0) {
                        const int nlo = qs > 0 ? lo + (int)(((int64_t)n * qs) / (G + 1)) + 1 : lo;
                        hi = lo + (int)(((int64_t)n * (qs + 1)) / (G + 1));
                        lo = nlo;
                    } else {
                        lo = lo + (int)(((int64_t)n * G) / (G + 1)) + 1;
                    }
                }
                if (!__syncthreads_or(active && hi > lo)) break;
            }
        }
        // x = lo: A keeps [.., x), B takes [x, ..)
        if (active) sm.cut[s] = inB ? max(sm.cut[s], lo) : min(sm.cut[s], lo);
        __syncthreads();
    }

    // ---- 3. fill this thread's columns ----
    if (!active) return;
    const int c0 = s * L, c1 = min(c0 + L, W);
    if (c0 >= W) return;
    int sg = owner_seg(sm, 0, T, c0);
    int seg_end = sg + 1 < T ? sm.cut[sg + 1] : W;
    int n = sm.cnt[sg];
    const uint32_t* st = sm.stk + sg * (L + 1);
    int e = 0;
    auto locate = [&](int j) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int)(st[mid] >> 16) <= j) lo = mid; else hi = mid - 1;
        }
        e = lo;
    };
    if (n > 0) locate(c0);
    uint32_t k = 0, rr = kNoRow, gk = kInfU;
    int next_start = W;
    auto load_entry = [&]() {
        if (n == 0) { k = 0; rr = kNoRow; gk = kInfU; next_start = W; return; }
        const uint32_t ent = st[e];
        k = ent & 0xffffu;
        rr = sm.nrs[nidx((int)k, L)];
        const uint32_t av = i > rr ? i - rr : rr - i;
        gk = av * av;
        next_start = e + 1 < n ? (int)(st[e + 1] >> 16) : W;
    };
    load_entry();

    int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + img * a.sD) + (int64_t)i * W : nullptr;
    float* Srow = a.S ? reinterpret_cast<float*>(a.S + img * a.sS) + (int64_t)i * W : nullptr;
    int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + img * a.sL) + (int64_t)i * W : nullptr;
    int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + img * a.sN) + (int64_t)i * W : nullptr;

    auto cell = [&](int j, int32_t& d, int32_t& lab, int32_t& col) {
        if (j >= seg_end) {
            while (sg + 1 < T && sm.cut[sg + 1] <= j) ++sg;
            seg_end = sg + 1 < T ? sm.cut[sg + 1] : W;
            n = sm.cnt[sg];
            st = sm.stk + sg * (L + 1);
            if (n > 0) locate(j);
            load_entry();
        }
        while (j >= next_start) {
            ++e;
            load_entry();
        }
        if (gk == kInfU) {
            d = DFC_INF_I32; lab = -1; col = -1;
        } else {
            const int dj = j - (int)k;
            d = (int32_t)(gk + (uint32_t)(dj * dj));
            lab = (int32_t)(rr * (uint32_t)W + k);
            col = (int32_t)k;
        }
    };

    if (a.vec) {
        for (int j = c0; j < c1; j += 4) {
            int4 d4, l4, n4;
            cell(j + 0, d4.x, l4.x, n4.x);
            cell(j + 1, d4.y, l4.y, n4.y);
            cell(j + 2, d4.z, l4.z, n4.z);
            cell(j + 3, d4.w, l4.w, n4.w);
            if (Drow) __stcs(reinterpret_cast<int4*>(Drow + j), d4);
            if (Srow) {
                const float4 f4 = make_float4(dist_f32(d4.x), dist_f32(d4.y), dist_f32(d4.z),
                                              dist_f32(d4.w));
                __stcs(reinterpret_cast<float4*>(Srow + j), f4);
            }
            if (Lrow) __stcs(reinterpret_cast<int4*>(Lrow + j), l4);
            if (Nrow) __stcs(reinterpret_cast<int4*>(Nrow + j), n4);
        }
    } else {
        for (int j = c0; j < c1; ++j) {
            int32_t d, lab, col;
            cell(j, d, lab, col);
            if (Drow) Drow[j] = d;
            if (Srow) Srow[j] = dist_f32((uint32_t)d);
            if (Lrow) Lrow[j] = lab;
            if (Nrow) Nrow[j] = col;
        }
    }
}

template __global__ void k_rows<false>(RowArgs);
template __global__ void k_rows<true>(RowArgs);

}  // namespace dfc
