// k_rows_win.cu -- stage 2 of the separable EDT without a merge tree: the
// per-row lower envelope of D_k(j) = g_k + (j-k)^2, g_k = (i - nearest_row_k)^2,
// evaluated by a bounded outward search over segment stacks.
//
// Replaces envelope_rows / build_row_envelope / meijster_scan
// (exact_edt.cpp:190-283) and the label assembly of voronoi_labels
// (exact_edt.cpp:362-369), like k_rows.cu, with a different stage 2b:
//
//  1. build   one thread per segment of L columns runs the reference stack
//             algorithm (Meijster, exact integer boundaries,
//             exact_edt.cpp:200-223) over its own columns, read straight
//             from HBM into registers: the envelope of the segment's
//             parabolas over the whole row [0, cols), kept in shared memory.
//  2. search  each thread evaluates the envelope of its OWN segment at its L
//             columns, then the stacks of other segments, nearest first
//             (alternating left/right), keeping the best (D, owner) per
//             column in registers.  A segment whose columns are all farther
//             than sqrt(Umax) from every column of the thread -- Umax = the
//             largest current D over its columns -- cannot own any of them:
//             the search stops on each side at the first such segment and
//             skips a segment whose (min g + gap^2) bound exceeds Umax.  The
//             result is exact: every minimiser k of column j has
//             (j-k)^2 <= D(j) <= Umax.
//  3. write   D, sqrt(D), the label and/or the nearest column, 16-byte
//             streaming stores.
//
// No barrier after the build, no merge bookkeeping: the work of a thread is
// its build plus one pass over its columns per segment within reach, which is
// a handful on the C1/C2/C4 images (dense features) and only grows where the
// nearest feature is far -- and there most segments are empty and skipped
// through a bitmask of non-empty segments.
//
// Tie rules are exact by processing order.  Inside a stack they are the
// reference's (keep_old: floor(x)+1 boundaries; take_new: ceil(x)).  Across
// stacks: every segment evaluated after the thread's own one lies farther
// out, so a LEFT segment has a smaller column than everything seen so far and
// a RIGHT one a larger column.  keep_old (smaller column wins, the label rule,
// exact_edt.cpp:205/:363) therefore lets left segments win ties (<=) and
// right segments only strictly (<); take_new (meijster_scan's nearest_col,
// exact_edt.cpp:275) the other way round.
//
// All arithmetic is exact 32-bit integer: every value is bounded by
// (rows-1)^2 + (cols-1)^2 <= 2^31-2 (DFC_MAX_SQDIST, SURVEY.md finding 7).
#include "dfc_kernels.cuh"

namespace dfc {

// Geometry of the window kernel: nseg = T * spt segments of L columns per row
// (a power of two >= ceil(cols / L)), T threads per row (<= 256), spt segments
// per thread, R rows per CTA.
struct WinLayout {
    int nseg, spt, lg;  // lg = log2(nseg)
};

// Shared memory per row (32-bit words): stack entries (column | start << 16),
// stack rows (uint16), staged nearest rows, per-segment {min g, first|last
// candidate}, count, non-empty bitmask.  Even, so uint2 arrays stay aligned.
__host__ __device__ __forceinline__ int win_meta_off(int nseg, int L) {
    const int ent = nseg * (L + 1);
    return (ent + (ent + 1) / 2 + nseg * (L / 2 + 1) + 1) & ~1;
}
inline int win_row_words(int nseg, int L) {
    return (win_meta_off(nseg, L) + 4 * nseg + (nseg + 31) / 32 + 1) & ~1;
}

__device__ __forceinline__ uint32_t st_first(const uint32_t* stk, int sg, int L) {
    return stk[sg * (L + 1)] & 0xffffu;
}

__device__ __forceinline__ int win_next_nz(const uint32_t* nzw, int x, int nseg) {
    if (x >= nseg) return nseg;
    int w = x >> 5;
    uint32_t m = nzw[w] & (0xffffffffu << (x & 31));
    const int nw = (nseg + 31) >> 5;
    while (m == 0) {
        if (++w >= nw) return nseg;
        m = nzw[w];
    }
    return (w << 5) + __ffs(m) - 1;
}

__device__ __forceinline__ int win_prev_nz(const uint32_t* nzw, int x) {
    if (x < 0) return -1;
    int w = x >> 5;
    uint32_t m = nzw[w] & (0xffffffffu >> (31 - (x & 31)));
    while (m == 0) {
        if (--w < 0) return -1;
        m = nzw[w];
    }
    return (w << 5) + 31 - __clz(m);
}

__device__ __forceinline__ uint32_t win_g(uint32_t gi, uint32_t r) {
    const uint32_t a = gi > r ? gi - r : r - gi;
    return a * a;
}

// Evaluate the stack of segment `st` (n entries, column | start << 16) at the
// warp's 32 columns c0 + lane and fold it into the lane's best.  The owner
// of column j is the last entry with start <= j: lanes hold one entry each,
// a ballot counts the entries starting at or before c0 and an OR-reduction
// marks those starting inside the window, so the owner index of lane x is a
// popcount; one shuffle fetches it.  SIDE: 0 = the warp's own segment (first,
// assigns), -1 = a segment to the left, +1 = to the right (tie rule above).
template <int SIDE, bool TAKE_NEW>
__device__ __forceinline__ void win_eval(const uint32_t* st, const uint16_t* sr, int n, int c0, int lane,
                                         uint32_t gi, uint32_t& bD, uint32_t& bP) {
    const bool valid = lane < n;
    const uint32_t ent = valid ? st[lane] : 0xffffffffu;  // invalid: start 0xFFFF > every column
    const uint32_t pk = (ent & 0xffffu) | (valid ? (uint32_t)sr[lane] << 16 : 0u);
    const int start = (int)(ent >> 16);
    const int nle = __popc(__ballot_sync(0xffffffffu, start <= c0));
    const uint32_t bit = (start > c0 && start < c0 + 32) ? (1u << (start - c0)) : 0u;
    const uint32_t inside = __reduce_or_sync(0xffffffffu, bit);
    const int own = nle - 1 + __popc(inside & ((2u << lane) - 1u));
    const uint32_t po = __shfl_sync(0xffffffffu, pk, own);
    const int dj = c0 + lane - (int)(po & 0xffffu);
    const uint32_t d = win_g(gi, po >> 16) + (uint32_t)(dj * dj);
    bool win;
    if (SIDE == 0) win = true;
    else if ((SIDE < 0) != TAKE_NEW) win = d <= bD;
    else win = d < bD;
    if (win) {
        bD = d;
        bP = po;
    }
}

template <bool TAKE_NEW>
__global__ void __launch_bounds__(256) k_rows_win(RowArgs a, WinLayout wl) {
    constexpr int L = 32;
    extern __shared__ uint32_t smem[];
    const int nseg = wl.nseg, lg = wl.lg;
    const int R = a.R;
    const int lane = threadIdx.x & 31;
    const int W = a.W;
    const int ent = nseg * (L + 1);
    auto row_of = [&](int rho, int& img, uint32_t& i) -> bool {
        const int64_t row = (int64_t)blockIdx.x * R + rho;
        if (row >= a.total_rows) return false;
        if (a.total_rows < (1ll << 31)) {
            img = (int)((uint32_t)row / (uint32_t)a.H);
            i = (uint32_t)row - (uint32_t)img * (uint32_t)a.H;
        } else {
            img = (int)(row / a.H);
            i = (uint32_t)(row - (int64_t)img * a.H);
        }
        return true;
    };

    // ---- 1. per-segment stacks (exact_edt.cpp:208-223): thread -> (row, segment) ----
    for (int p = threadIdx.x; p < R * nseg; p += blockDim.x) {  // trip count uniform per CTA
        const int rho = p >> lg, sg = p & (nseg - 1);
        int img = 0;
        uint32_t i = 0;
        const bool active = row_of(rho, img, i);
        const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;
        uint32_t* base = smem + rho * a.row_smem_words;
        uint32_t* stk = base;                                              // [nseg][L+1]
        uint16_t* srr = reinterpret_cast<uint16_t*>(base + ent);           // [nseg][L+1]
        uint32_t* nrw = base + ent + (ent + 1) / 2;                        // [nseg][L/2+1] staged nr pairs
        uint2* meta = reinterpret_cast<uint2*>(base + win_meta_off(nseg, L));  // [nseg] {min g, first | last << 16}
        int* cnt = reinterpret_cast<int*>(meta + nseg);                    // [nseg]
        uint32_t* nzw = reinterpret_cast<uint32_t*>(cnt + nseg);           // [ceil(nseg/32)]
        const uint16_t* rowp = a.nr + img * a.nr_img_stride + (int64_t)i * a.Wp;
        const int c0 = sg * L, c1 = min(c0 + L, W);
        int n = 0;
        uint32_t gmin = kInfU;
        if (active && c0 < W) {
            // stage this segment's nearest rows: 16-byte loads -> the thread's own words
            uint32_t* mine = nrw + sg * (L / 2 + 1);
            const int tl = a.tile_cols >= W ? 0 : c0 / a.tile_cols;
            const uint16_t* q16 = rowp + tl * a.tile_stride + (c0 - tl * a.tile_cols);
            if (a.vec_nr && c0 + L <= W) {
                const uint4* q = reinterpret_cast<const uint4*>(q16);
#pragma unroll
                for (int u = 0; u < L / 8; ++u) {
                    const uint4 w4 = __ldg(q + u);
                    mine[4 * u + 0] = w4.x;
                    mine[4 * u + 1] = w4.y;
                    mine[4 * u + 2] = w4.z;
                    mine[4 * u + 3] = w4.w;
                }
            } else {
                for (int u = 0; u < L / 2; ++u) {
                    uint32_t lo = kNoRow, hi = kNoRow;
                    const int j0 = c0 + 2 * u;
                    if (j0 < W) {
                        const int t0 = a.tile_cols >= W ? 0 : j0 / a.tile_cols;
                        lo = __ldg(rowp + t0 * a.tile_stride + (j0 - t0 * a.tile_cols));
                    }
                    if (j0 + 1 < W) {
                        const int t1 = a.tile_cols >= W ? 0 : (j0 + 1) / a.tile_cols;
                        hi = __ldg(rowp + t1 * a.tile_stride + (j0 + 1 - t1 * a.tile_cols));
                    }
                    mine[u] = lo | (hi << 16);
                }
            }
            const uint16_t* nrs = reinterpret_cast<const uint16_t*>(mine);
            uint32_t* st = stk + sg * (L + 1);
            uint16_t* sr = srr + sg * (L + 1);
            int tk = 0, ts = 0;
            uint32_t tg = 0;
            // One event per iteration -- pop the top, or consume column m (push
            // or skip) -- so the lanes of a warp reconverge every iteration.
            int m = c0;
            uint32_t rm = nrs[0];
            while (m < c1) {
                if (rm == kNoRow) {
                    ++m;
                    rm = m < c1 ? nrs[m - c0] : kNoRow;
                    continue;
                }
                const uint32_t gm = win_g(gi, rm);
                bool consume = true;
                int start = 0;
                bool push = true;
                if (n > 0) {
                    if (gm == 0 && tg == 0 && tk == m - 1) {
                        // run of object pixels: the zero parabola starts at m, pops nothing
                        start = m;
                    } else {
                        // num = g_m - g_k + m^2 - k^2 fits int32; ts * den < 2^32
                        const int num = (int)gm - (int)tg + (m * m - tk * tk);
                        const uint32_t den = 2u * (uint32_t)(m - tk);
                        const uint32_t lim = (uint32_t)ts * den;  // start <= js[idx]  (:214)
                        if (num < 0 || (TAKE_NEW ? (uint32_t)num <= lim : (uint32_t)num < lim)) {
                            consume = false;  // pop
                            if (--n > 0) {
                                const uint32_t e = st[n - 1];
                                tk = (int)(e & 0xffffu);
                                ts = (int)(e >> 16);
                                tg = win_g(gi, sr[n - 1]);
                            }
                        } else {
                            // push iff start <= cols-1 (:218)
                            const uint32_t lim2 = (uint32_t)(W - 1) * den;
                            push = TAKE_NEW ? (uint32_t)num <= lim2 : (uint32_t)num < lim2;
                            const uint32_t qd = small_udiv((uint32_t)num, den);
                            // keep_old: floor(x)+1 ; take_new: ceil(x)   (:205)
                            start = TAKE_NEW ? (int)(qd + ((uint32_t)num != qd * den)) : (int)qd + 1;
                        }
                    }
                }
                if (consume) {
                    if (push) {
                        st[n] = (uint32_t)m | ((uint32_t)start << 16);
                        sr[n] = (uint16_t)rm;
                        ++n;
                        tk = m;
                        ts = start;
                        tg = gm;
                        gmin = min(gmin, gm);
                    }
                    ++m;
                    rm = m < c1 ? nrs[m - c0] : kNoRow;
                }
            }
        }
        if (active) {
            cnt[sg] = n;
            meta[sg] = make_uint2(gmin, n > 0 ? ((st_first(stk, sg, L)) | ((stk[sg * (L + 1) + n - 1] & 0xffffu) << 16)) : 0u);
        }
        // non-empty bitmask: one word per 32 consecutive segments of a row
        const uint32_t bal = __ballot_sync(0xffffffffu, n > 0);
        if (nseg >= 32) {
            if (lane == 0 && active) nzw[sg >> 5] = bal;
        } else if (sg == 0 && active) {
            nzw[0] = (bal >> (lane & ~(nseg - 1) & 31)) & (nseg == 32 ? 0xffffffffu : ((1u << nseg) - 1u));
        }
    }
    __syncthreads();

    // ---- 2. outward search, one warp per segment, lane = column ----
    const int warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    int cur_rho = -1, img = 0;
    uint32_t i = 0;
    bool row_ok = false;
    for (int p = warp; p < R * nseg; p += nwarp) {
        const int rho = p >> lg, sg = p & (nseg - 1);
        if (rho != cur_rho) {
            cur_rho = rho;
            row_ok = row_of(rho, img, i);
        }
        const int c0 = sg * L;
        if (!row_ok || c0 >= W) continue;  // warp-uniform
        const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;
        const uint32_t* base = smem + rho * a.row_smem_words;
        const uint32_t* stk = base;
        const uint16_t* srr = reinterpret_cast<const uint16_t*>(base + ent);
        const uint2* meta = reinterpret_cast<const uint2*>(base + win_meta_off(nseg, L));
        const int* cnt = reinterpret_cast<const int*>(meta + nseg);
        const uint32_t* nzw = reinterpret_cast<const uint32_t*>(cnt + nseg);
        const int j = c0 + lane;
        const bool live = j < W;

        uint32_t bD = kInfU, bP = 0;
        const int n0 = cnt[sg];
        if (n0 > 0) win_eval<0, TAKE_NEW>(stk + sg * (L + 1), srr + sg * (L + 1), n0, c0, lane, gi, bD, bP);
        int pl = win_prev_nz(nzw, sg - 1), pr = win_next_nz(nzw, sg + 1, nseg);
        while (true) {
            // a side ends at the first segment none of whose columns is within
            // sqrt(D) of a column of this warp (every later one is farther)
            if (pl >= 0) {
                const int dl = j - (pl * L + L - 1);
                if (!__any_sync(0xffffffffu, live && (uint32_t)(dl * dl) <= bD)) pl = -1;
            }
            if (pr < nseg) {
                const int dr = pr * L - j;
                if (!__any_sync(0xffffffffu, live && (uint32_t)(dr * dr) <= bD)) pr = nseg;
            }
            if (pl < 0 && pr >= nseg) break;
            const bool goL = pl >= 0 && (pr >= nseg || sg - pl <= pr - sg);
            const int s2 = goL ? pl : pr;
            const uint2 mt = meta[s2];
            // nearest candidate of that segment to column j, with its smallest g
            const int dk = j - (int)(goL ? (mt.y >> 16) : (mt.y & 0xffffu));
            if (__any_sync(0xffffffffu, live && mt.x + (uint32_t)(dk * dk) <= bD)) {
                if (goL) win_eval<-1, TAKE_NEW>(stk + s2 * (L + 1), srr + s2 * (L + 1), cnt[s2], c0, lane, gi, bD, bP);
                else win_eval<1, TAKE_NEW>(stk + s2 * (L + 1), srr + s2 * (L + 1), cnt[s2], c0, lane, gi, bD, bP);
            }
            if (goL) pl = win_prev_nz(nzw, pl - 1);
            else pr = win_next_nz(nzw, pr + 1, nseg);
        }

        // ---- 3. write: lane x -> column c0 + x (coalesced) ----
        if (!live) continue;
        const int64_t off = (int64_t)i * W + j;
        const bool inf = bD == kInfU;
        if (a.D) __stcs(reinterpret_cast<int32_t*>(a.D + img * a.sD) + off, inf ? DFC_INF_I32 : (int32_t)bD);
        if (a.S) __stcs(reinterpret_cast<float*>(a.S + img * a.sS) + off, dist_f32(bD));
        if (a.LB)
            __stcs(reinterpret_cast<int32_t*>(a.LB + img * a.sL) + off,
                   inf ? -1 : (int32_t)((bP >> 16) * (uint32_t)W + (bP & 0xffffu)));
        if (a.NC) __stcs(reinterpret_cast<int32_t*>(a.NC + img * a.sN) + off, inf ? -1 : (int32_t)(bP & 0xffffu));
    }
}

template <bool TAKE_NEW>
inline const void* win_kernel_ptr() {
    return (const void*)k_rows_win<TAKE_NEW>;
}

}  // namespace dfc
