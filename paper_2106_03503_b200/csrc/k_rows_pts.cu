// k_rows_pts.cu -- stage 2 for POINT planes: at most kPtsCap object pixels
// (C3's 30-point images).
//
// Same result as k_rows.cu / k_rows_lr.cu (envelope_rows / meijster_scan /
// voronoi label assembly, exact_edt.cpp:190-283, :362-369), without the
// nearest-row plane: K1a (k_columns.cu) already listed the plane's object
// pixels, so K1b/K1c skip the plane and this kernel reads only that list.
//
//  list    one warp = 32 rows of one plane (rows per plane a multiple of 32).
//          The warp sorts the plane's <= kPtsCap (32) keys (column << 16 | row)
//          by rank counting (keys are distinct pixels) and compacts the distinct
//          object columns with their row ranges.
//  build   lane = row i: for every object column k in order, the nearest object
//          row of that column (binary search in the column's sorted rows; the
//          upper row on a tie, as the reference's fused vertical pass,
//          exact_edt.cpp:351) gives g_k; the reference's stack algorithm
//          (exact_edt.cpp:208-223, exact integer boundaries, keep_old or
//          take_new) over the <= kPtsCap candidates builds the row's whole
//          envelope in shared memory.  Columns without an object never enter
//          the envelope (:212).
//  fill    the shared lr_fill_row (k_rows_lr.cu): lane = column, 128-column
//          blocks, 16-byte stores.
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kPtsWarps = 4;  // ~8.6 KB of static shared memory per warp
constexpr int kPtsStride = kPtsCap + 1;  // words per row's envelope (odd: conflict-free)

struct PtsSmem {
    uint32_t key[kPtsCap];               // sorted keys
    uint16_t ucol[kPtsCap];              // distinct object columns
    uint16_t ubeg[kPtsCap + 1];          // their ranges in key[]
    uint32_t ks[32][kPtsStride];         // per row: envelope entries column | start << 16
    uint16_t rr[32][2 * kPtsStride];     // per row: the entries' nearest rows
};

template <bool TAKE_NEW>
__global__ void __launch_bounds__(32 * kPtsWarps) k_rows_pts(RowArgs a, const uint32_t* __restrict__ pts) {
    __shared__ PtsSmem smem[kPtsWarps];
    PtsSmem& sm = smem[threadIdx.x >> 5];
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int W = a.W;
    const int64_t band = (int64_t)blockIdx.x * kPtsWarps + (threadIdx.x >> 5);
    if (band * 32 >= a.total_rows) return;
    const int img = (int)(band * 32 / a.H);  // the whole warp: rows per plane % 32 == 0
    if (!pts_plane(a.plane_counts, img, a.pts_gate)) return;
    const int n = (int)a.plane_counts[img];
    const uint32_t i = (uint32_t)(band * 32 + lane - (int64_t)img * a.H);

    // ---- sort the plane's keys (rank = number of smaller keys) ----
    const uint32_t* src = pts + (int64_t)img * kPtsCap;
    static_assert(kPtsCap <= 32, "one key per lane");
    const uint32_t k0 = lane < n ? __ldg(src + lane) : FULL;
    int rank0 = 0;
    for (int q = 0; q < n; ++q) rank0 += __shfl_sync(FULL, k0, q) < k0;
    if (lane < n) sm.key[rank0] = k0;
    __syncwarp();
    // ---- distinct columns: a key starts a column when its column differs ----
    int nu = 0;
    for (int q0 = 0; q0 < n; q0 += 32) {
        const int q = q0 + lane;
        const bool head = q < n && (q == 0 || (sm.key[q] >> 16) != (sm.key[q - 1] >> 16));
        const unsigned m = __ballot_sync(FULL, head);
        if (head) {
            const int u = nu + __popc(m & ((1u << lane) - 1u));
            sm.ucol[u] = (uint16_t)(sm.key[q] >> 16);
            sm.ubeg[u] = (uint16_t)q;
        }
        nu += __popc(m);
    }
    if (lane == 0) sm.ubeg[nu] = (uint16_t)n;
    __syncwarp();

    // ---- the row's envelope over the object columns (exact_edt.cpp:208-223) ----
    uint32_t* st = sm.ks[lane];
    uint16_t* sr = sm.rr[lane];
    int ns = 0, tk = 0, ts = 0;
    uint32_t tg = 0;
    for (int u = 0; u < nu; ++u) {
        const int m = sm.ucol[u];
        // nearest object row of column m: first row >= i, and the one before it
        int lo = sm.ubeg[u], hi = sm.ubeg[u + 1];
        const int b0 = lo;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((sm.key[mid] & 0xffffu) < i) lo = mid + 1;
            else hi = mid;
        }
        const uint32_t rb = lo < sm.ubeg[u + 1] ? (sm.key[lo] & 0xffffu) : kNoRow;
        const uint32_t ra = lo > b0 ? (sm.key[lo - 1] & 0xffffu) : kNoRow;
        const uint32_t r = pick_nearest(i, ra, rb);  // upper row on a tie
        const uint32_t av = i > r ? i - r : r - i;
        const uint32_t gm = av * av;
        int start = 0;
        bool push = true;
        while (ns > 0) {
            // num = g_m - g_k + m^2 - k^2, |num| < 2^31; ts*den, (W-1)*den < 2^31
            const int dm = m - tk;
            const int num = (int)gm - (int)tg + dm * (m + tk);
            const int den = 2 * dm;
            if (TAKE_NEW ? num <= ts * den : num < ts * den) {  // start <= js[idx]: pop (:214)
                if (--ns > 0) {
                    const uint32_t e = st[ns - 1];
                    tk = (int)(e & 0xffffu);
                    ts = (int)(e >> 16);
                    const uint32_t rk = sr[ns - 1];
                    const uint32_t ak = i > rk ? i - rk : rk - i;
                    tg = ak * ak;
                }
                continue;
            }
            push = TAKE_NEW ? num <= (W - 1) * den : num < (W - 1) * den;  // start <= cols-1 (:218)
            if (push) {
                const uint32_t q = small_udiv((uint32_t)num, (uint32_t)den);
                start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * (uint32_t)den)) : (int)q + 1;  // (:205)
            }
            break;
        }
        if (!push) continue;
        st[ns] = (uint32_t)m | ((uint32_t)start << 16);
        sr[ns] = (uint16_t)r;
        ++ns;
        tk = m;
        ts = start;
        tg = gm;
    }
    if (ns == 0) {  // featureless plane: every cell infinite (test_exact_edt.cpp:223-227)
        st[0] = kLrInfK;
        sr[0] = kNoRow;
        ns = 1;
    }
    __syncwarp();

    // ---- fill, row by row ----
    for (int rho = 0; rho < 32; ++rho) {
        const int nE = __shfl_sync(FULL, ns, rho);
        const uint32_t giR = __shfl_sync(FULL, i, rho);
        const int64_t rowR = band * 32 + rho;
        const int64_t iR = rowR - (int64_t)img * a.H;
        int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + img * a.sD) + iR * W : nullptr;
        float* Srow = a.S ? reinterpret_cast<float*>(a.S + img * a.sS) + iR * W : nullptr;
        int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + img * a.sL) + iR * W : nullptr;
        int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + img * a.sN) + iR * W : nullptr;
        lr_fill_row(a, sm.ks[rho], sm.rr[rho], nE, giR, Drow, Srow, Lrow, Nrow, 0, W, lane);
    }
}

template <bool TAKE_NEW>
inline const void* pts_kernel_ptr() {
    return (const void*)k_rows_pts<TAKE_NEW>;
}

}  // namespace dfc
