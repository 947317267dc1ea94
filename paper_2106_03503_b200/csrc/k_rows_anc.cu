// k_rows_anc.cu -- stage 2 as ANCHORED SEGMENTS: one CTA per row, anchors by
// divide and conquer, then a uniform brute-force pass per 32-column segment.
//
// Same result as k_rows.cu (envelope_rows / meijster_scan / voronoi label
// assembly, exact_edt.cpp:190-283, :362-369), different decomposition.  The
// reference builds the lower envelope of the parabolas D_k(j) = g_k + (j-k)^2
// with a stack (exact_edt.cpp:208-223); its owners (the smallest minimiser
// under keep_old, the largest under take_new, :205/:275) are monotone in j.
// This kernel uses only that monotonicity:
//
//  stage    the row's vertical values g_k = (i - nr_k)^2 (kAncInf: no object
//           in column k, :212) go to the CTA's shared memory once.
//  anchors  owner(32 s) for every segment s, by divide and conquer over s:
//           owner(32 s) lies in [owner(32 s_lo), owner(32 s_hi)] for any
//           computed s_lo < s < s_hi (bounds: the first / last finite column).
//           Each anchor is a warp-parallel scan of its candidate range (lane =
//           candidate, the tie rule within a lane by scan order) and a REDUX
//           min over the values, then min / max over the columns attaining it.
//           The ranges of one level overlap only at their ends, so a level
//           costs about W/32 warp iterations.
//  segments lane = column j of segment [32 s, 32 s + 32): brute force over the
//           candidates [owner(32 s), owner(32 s + 32)] (owner(W) := the last
//           finite column) in increasing order, keep_old updating on <,
//           take_new on <=.  Every iteration is warp-uniform: no divergence,
//           no stack, and the ranges of a row sum to about W + W/32.
//
// A row with no finite g is written as featureless (D = DFC_INF_I32).
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kAncWarps = 4;               // warps per CTA (one row per CTA)
constexpr int kAncMaxW = 16384;
// Shared memory holds h_k = g_k + k^2 (int32), so that D_k(j) - j^2 = h_k - 2 j k
// is one multiply-add (or, with 2 j k carried along, one 3-way add).  A column
// without objects gets g = kAncInf = kAncBig^2: above every real D (rows <= 32768,
// columns <= kAncMaxW: D <= 32767^2 + 16383^2 < 1.35e9 < 1.6e9), and h,
// h - 2jk stay inside int32.
constexpr uint32_t kAncBig = 40000;  // vertical distance of a column without objects
constexpr int32_t kAncInf = (int32_t)(kAncBig * kAncBig);

__host__ __device__ __forceinline__ int anc_segs(int W) { return (W + 31) >> 5; }
// words: g (W, 16-byte granules), anchors (S + 1), per-warp partial owners (2 NW),
// object-pixel bits of the row (S)
__host__ __device__ __forceinline__ int anc_gwords(int W) { return (W + 3) & ~3; }
inline int anc_smem_bytes(int W) { return (anc_gwords(W) + 2 * anc_segs(W) + 1 + 2 * kAncWarps) * 4; }

// The rows this kernel owns in the default row pass: not a point plane; in a
// sparse plane (k_rows_lr) only the rows that kernel flagged (2); elsewhere the
// rows k_rows_dense did not write (1).
__device__ __forceinline__ bool anc_row_mine(const RowArgs& a, int64_t row, int img) {
    if (pts_plane(a.plane_counts, img, a.pts_gate)) return false;
    const uint8_t rd = a.row_done ? a.row_done[row] : 0;
    if (a.lr_gate && lr_plane(a.plane_counts, img, a.H, a.W)) return rd == 2;
    return rd != 1;
}

constexpr int32_t kAncNone = 0x7FFFFFFF;  // "no candidate" (empty range)

// Minimum of D_k(j) - j^2 = h_k - 2 j k over the candidates [lo, hi] (possibly
// empty: kAncNone) and the column attaining it: lane = candidate, ascending per
// lane (two candidates per step); then a REDUX min over the values and, among
// the lanes attaining it, the smallest (keep_old) or largest (take_new) column.
template <bool TAKE_NEW>
__device__ __forceinline__ int32_t anc_owner(const int32_t* h, int j, int lo, int hi, int lane, int& col) {
    int32_t best = kAncNone;
    int bk = lo;
    const int c = -2 * j;
    int k = lo + lane;
    for (; k + 32 <= hi; k += 64) {
        const int32_t v0 = h[k] + c * k, v1 = h[k + 32] + c * (k + 32);
        if (TAKE_NEW ? v0 <= best : v0 < best) {
            best = v0;
            bk = k;
        }
        if (TAKE_NEW ? v1 <= best : v1 < best) {
            best = v1;
            bk = k + 32;
        }
    }
    if (k <= hi) {
        const int32_t v0 = h[k] + c * k;
        if (TAKE_NEW ? v0 <= best : v0 < best) {
            best = v0;
            bk = k;
        }
    }
    const int32_t m = __reduce_min_sync(0xffffffffu, best);
    col = TAKE_NEW ? (int)__reduce_max_sync(0xffffffffu, best == m ? (uint32_t)bk : 0u)
                   : (int)__reduce_min_sync(0xffffffffu, best == m ? (uint32_t)bk : 0xFFFFFFFFu);
    return m;
}

template <bool TAKE_NEW, bool OWNERS>
__global__ void __launch_bounds__(32 * kAncWarps) k_rows_anc(RowArgs a) {
    extern __shared__ uint4 ancsm[];
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int NW = kAncWarps;
    const int W = a.W;
    const int S = anc_segs(W);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int32_t* g = reinterpret_cast<int32_t*>(ancsm);         // h_k = g_k + k^2
    int* anc = reinterpret_cast<int*>(g + anc_gwords(W));  // [S + 1]
    int32_t* pv = reinterpret_cast<int32_t*>(anc + S + 1);  // [NW] partial minima
    int* pk = reinterpret_cast<int*>(pv + NW);                // [NW] their columns
    uint32_t* zb = reinterpret_cast<uint32_t*>(pk + NW);      // [S] bit = object pixel on the row
    int P = 1;                                                // power of two >= S
    while (P < S) P <<= 1;

    // all rows (skipping the ones other kernels own), or a compact list of them
    const int64_t nrows = a.row_list ? (int64_t)*a.row_count : a.total_rows;
    for (int64_t q = blockIdx.x; q < nrows; q += gridDim.x) {
        const int64_t row = a.row_list ? (int64_t)a.row_list[q] : q;
        const int img = (int)(row / a.H);
        if (!a.row_list && !anc_row_mine(a, row, img)) continue;  // CTA-uniform
        const uint32_t i = (uint32_t)(row - (int64_t)img * a.H);
        const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;
        const uint16_t* rowp = a.nr + img * a.nr_img_stride + (int64_t)i * a.Wp;

        // ---- stage h = g + k^2, the row's object-pixel bits, and whether any
        // column is finite.  Thread = 4 consecutive columns; a column's vertical
        // distance d (kAncBig: no object in the column) comes from the nearest-row
        // plane or from the band's mask and carries (as K1c, k_columns.cu). ----
        const int bb = (int)(i >> 5), br = (int)(i & 31);
        const int slot = a.bmask ? img / a.n_img : 0;
        const int bpol = a.bpol0 + slot;
        const uint32_t bvalid = a.bmask && a.H - 32 * bb < 32 ? (1u << (a.H - 32 * bb)) - 1u : 0xffffffffu;
        const uint32_t upmask = 0xffffffffu >> (31 - br);
        const uint32_t* mrow = a.bmask ? a.bmask + ((int64_t)(img - slot * a.n_img) * a.nb + bb) * a.Wp : nullptr;
        const uint16_t* arow = a.bmask ? a.babove + ((int64_t)img * a.nb + bb) * a.Wp : nullptr;
        const uint16_t* brow = a.bmask ? a.bbelow + ((int64_t)img * a.nb + bb) * a.Wp : nullptr;
        // nearest object row (the upper one on a tie, exact_edt.cpp:351), for labels
        auto band_nr = [&](uint32_t m, uint32_t ca, uint32_t cb) -> uint32_t {
            const uint32_t mk = pol_mask(m, bpol, bvalid);
            const uint32_t up = mk & upmask, dn = mk >> br;
            const uint32_t ra = up ? (uint32_t)(32 * bb + 31 - __clz(up)) : ca;
            const uint32_t rb = dn ? (uint32_t)(i + __ffs(dn) - 1) : cb;
            return pick_nearest(i, ra, rb);
        };
        bool any = false;
        for (int q0 = warp * 32; 4 * q0 < W; q0 += 32 * NW) {  // warp-uniform trip count
            const int q = q0 + lane;
            const bool live = 4 * q < W;
            uint32_t d[4] = {kAncBig, kAncBig, kAncBig, kAncBig};
            if (live) {
                if (a.bmask) {
                    const uint4 m4 = __ldg(reinterpret_cast<const uint4*>(mrow) + q);
                    const uint2 a2 = __ldg(reinterpret_cast<const uint2*>(arow) + q);
                    const uint2 b2 = __ldg(reinterpret_cast<const uint2*>(brow) + q);
                    const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w};
                    const uint32_t ca[4] = {a2.x & 0xffffu, a2.x >> 16, a2.y & 0xffffu, a2.y >> 16};
                    const uint32_t cb[4] = {b2.x & 0xffffu, b2.x >> 16, b2.y & 0xffffu, b2.y >> 16};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint32_t mk = pol_mask(mm[t], bpol, bvalid);
                        const uint32_t up = mk & upmask, dn = mk >> br;
                        const uint32_t du = up ? (uint32_t)(br - 31) + __clz(up) : (ca[t] == kNoRow ? kAncBig : i - ca[t]);
                        const uint32_t dd = dn ? (uint32_t)__ffs(dn) - 1u : (cb[t] == kNoRow ? kAncBig : cb[t] - i);
                        d[t] = min(min(du, dd), kAncBig);
                    }
                } else {
                    uint32_t r[4];
                    if (a.vec_nr) {
                        const uint2 v = __ldg(reinterpret_cast<const uint2*>(rowp) + q);
                        r[0] = v.x & 0xffffu; r[1] = v.x >> 16; r[2] = v.y & 0xffffu; r[3] = v.y >> 16;
                    } else {
#pragma unroll
                        for (int t = 0; t < 4; ++t) r[t] = 4 * q + t < W ? (uint32_t)__ldg(rowp + 4 * q + t) : kNoRow;
                    }
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        d[t] = r[t] == kNoRow ? kAncBig : (gi > r[t] ? gi - r[t] : r[t] - gi);
                }
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (4 * q + t >= W) d[t] = kAncBig;  // padding past the row
            }
            int32_t o[4];
            uint32_t z = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = 4 * q + t;
                o[t] = (int32_t)(d[t] * d[t]) + j * j;
                any |= d[t] < kAncBig;
                z |= (uint32_t)(d[t] == 0 || j >= W) << t;
            }
            if (live) reinterpret_cast<int4*>(g)[q] = make_int4(o[0], o[1], o[2], o[3]);
            // object-pixel bits: 8 lanes x 4 columns = one 32-column word
            z <<= 4 * (lane & 7);
            z |= __shfl_xor_sync(FULL, z, 1);
            z |= __shfl_xor_sync(FULL, z, 2);
            z |= __shfl_xor_sync(FULL, z, 4);
            if ((lane & 7) == 0 && (q >> 3) < S) zb[q >> 3] = z;
        }
        // the owner search bounds are the row ends: a range containing columns
        // without objects still holds its finite owner, which beats them
        const int ff = 0, lf = W - 1;
        any = __syncthreads_or(any);

        int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + img * a.sD) + (int64_t)i * W : nullptr;
        float* Srow = a.S ? reinterpret_cast<float*>(a.S + img * a.sS) + (int64_t)i * W : nullptr;
        int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + img * a.sL) + (int64_t)i * W : nullptr;
        int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + img * a.sN) + (int64_t)i * W : nullptr;

        if (!any) {  // featureless row (CTA-uniform)
            for (int j = tid; j < W; j += 32 * NW) {
                if (Drow) __stcs(Drow + j, DFC_INF_I32);
                if (Srow) __stcs(Srow + j, __int_as_float(0x7f800000));
                if (Lrow) __stcs(Lrow + j, -1);
                if (Nrow) __stcs(Nrow + j, -1);
            }
            __syncthreads();
            continue;
        }

        // ---- anchors owner(32 s), s < S: levels of a divide and conquer over
        // [0, P] (index >= S stands for owner(W) := W - 1; index 0 comes last
        // with lower bound 0).  A level with n >= NW anchors gives each warp whole
        // anchors; with fewer, each anchor's range is split over NW / n warps
        // (ascending parts) and the parts are combined with the tie rule. ----
        if (tid == 0) anc[S] = lf;
        for (int step = P >> 1; step >= 0; step >>= 1) {
            const bool last = step == 0;  // anchor 0
            const int s0 = last ? 0 : step, ds = last ? 1 : 2 * step;
            const int n = last ? 1 : (S - step + ds - 1) >> (__ffs(ds) - 1);  // ds: a power of two
            if (n <= 0) continue;
            __syncthreads();
            auto bounds = [&](int s, int& lo, int& hi) {
                lo = (last || s - step == 0) ? ff : anc[s - step];
                hi = last ? (S > 1 ? anc[1] : lf) : (s + step >= S ? lf : anc[s + step]);
            };
            // an object pixel on the row owns itself (g = 0: the unique minimum)
            auto on_row = [&](int j) { return (zb[j >> 5] >> (j & 31)) & 1u; };
            if (n >= NW) {
                for (int t = warp; t < n; t += NW) {
                    const int s = s0 + t * ds;
                    int lo, hi, col = 32 * s;
                    if (!on_row(32 * s)) {
                        bounds(s, lo, hi);
                        anc_owner<TAKE_NEW>(g, 32 * s, lo, hi, lane, col);
                    }
                    if (lane == 0) anc[s] = col;
                }
            } else {
                const int q = NW / n;
                const int t = warp / q, part = warp - t * q;
                int32_t m = kAncNone;
                int col = 0;
                if (t < n) {
                    const int s = s0 + t * ds;
                    if (on_row(32 * s)) {
                        if (part == 0) {
                            m = -(32 * s) * (32 * s);
                            col = 32 * s;
                        }
                    } else {
                        int lo, hi;
                        bounds(s, lo, hi);
                        const int c = (hi - lo + q) / q;  // ceil((hi - lo + 1) / q)
                        const int plo = lo + part * c, phi = min(hi, plo + c - 1);
                        m = anc_owner<TAKE_NEW>(g, 32 * s, plo, phi, lane, col);
                    }
                }
                if (lane == 0) {
                    pv[warp] = m;
                    pk[warp] = col;
                }
                __syncthreads();
                if (tid < n) {
                    int32_t bm = kAncNone;
                    int bc = 0;
                    for (int p = 0; p < q; ++p) {  // ascending column ranges
                        const int32_t v = pv[tid * q + p];
                        if (TAKE_NEW ? (v <= bm && v != kAncNone) : v < bm) {
                            bm = v;
                            bc = pk[tid * q + p];
                        }
                    }
                    anc[s0 + tid * ds] = bc;
                }
            }
            if (last) break;
        }
        __syncthreads();

        // nearest object row of column k (labels): the plane, or the bands
        auto nr_of = [&](int k) -> uint32_t {
            if (!a.bmask) return (uint32_t)__ldg(rowp + k);
            return band_nr(__ldg(mrow + k), __ldg(arow + k), __ldg(brow + k));
        };

        // ---- segments: lane = column, brute force over [owner(j0), owner(j0 + 32)] ----
        for (int s = warp; s < S; s += NW) {
            const int j = 32 * s + lane;
            if (zb[s] == 0xffffffffu) {  // every column an object pixel on the row (warp-uniform)
                if (j < W) {
                    if (Drow) __stcs(Drow + j, 0);
                    if (Srow) __stcs(Srow + j, 0.0f);
                    if (OWNERS) {
                        if (Lrow) __stcs(Lrow + j, (int32_t)(nr_of(j) * (uint32_t)W + (uint32_t)j));
                        if (Nrow) __stcs(Nrow + j, j);
                    }
                }
                continue;
            }
            const int lo = anc[s], hi = anc[s + 1];
            // D_k(j) - j^2 = h_k - 2 j k, ascending k; the j^2 goes back at the end
            const int c = -2 * j;
            int32_t best;
            int bk = lo;
            if (OWNERS) {  // the minimiser too: one ordered scan (tie rule by order)
                best = kAncNone;
                int ck = c * lo;
#pragma unroll 4
                for (int k = lo; k <= hi; ++k, ck += c) {
                    const int32_t v = g[k] + ck;
                    if (TAKE_NEW ? v <= best : v < best) {
                        best = v;
                        bk = k;
                    }
                }
            } else {
                // the value only: running minima over the aligned superset
                // [lo & ~3, hi | 3] of the range (extra candidates cannot go
                // below the minimum, which the range attains; the padding past
                // W holds kAncInf + k^2), 16-byte loads of h
                int32_t b0 = kAncNone, b1 = b0;
                const int c2 = 2 * c, c3 = 3 * c;
                int k = lo & ~3;
                for (; k + 4 <= hi; k += 8) {
                    const int4 q = *reinterpret_cast<const int4*>(g + k);
                    const int4 r = *reinterpret_cast<const int4*>(g + k + 4);
                    const int ck = c * k, ck4 = ck + 2 * c2;
                    b0 = min(b0, min(q.x + ck, q.y + (ck + c)));
                    b1 = min(b1, min(q.z + (ck + c2), q.w + (ck + c3)));
                    b0 = min(b0, min(r.x + ck4, r.y + (ck4 + c)));
                    b1 = min(b1, min(r.z + (ck4 + c2), r.w + (ck4 + c3)));
                }
                if (k <= hi) {
                    const int4 q = *reinterpret_cast<const int4*>(g + k);
                    const int ck = c * k;
                    b0 = min(b0, min(q.x + ck, q.y + (ck + c)));
                    b1 = min(b1, min(q.z + (ck + c2), q.w + (ck + c3)));
                }
                best = min(b0, b1);
            }
            const uint32_t dval = (uint32_t)(best + j * j);
            if (j < W) {
                if (Drow) __stcs(Drow + j, (int32_t)dval);
                if (Srow) __stcs(Srow + j, dist_f32(dval));
                if (OWNERS) {
                    if (Lrow) __stcs(Lrow + j, (int32_t)(nr_of(bk) * (uint32_t)W + (uint32_t)bk));
                    if (Nrow) __stcs(Nrow + j, bk);
                }
            }
        }
        __syncthreads();
    }
}

template <bool TAKE_NEW, bool OWNERS>
inline const void* anc_kernel_ptr() {
    return (const void*)k_rows_anc<TAKE_NEW, OWNERS>;
}

}  // namespace dfc
