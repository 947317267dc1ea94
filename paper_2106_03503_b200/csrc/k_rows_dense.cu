// k_rows_dense.cu -- stage 2 for DENSE rows: rows whose object pixels (on the
// row itself) leave only short runs of other columns.
//
// On row i a column k with an object pixel ON the row (nearest row == i, g = 0)
// owns itself: D = 0 is the unique minimum.  For any other column j, let z1 <
// j < z2 be the nearest such columns (or the row ends): every candidate k < z1
// has D_k(j) = g_k + (j-k)^2 > (j-z1)^2 = D_z1(j) (and symmetrically beyond
// z2), strictly, so the owner of j -- under either tie rule -- is a column of
// [z1, z2].  When every run (z1, z2) is short, one warp per row evaluates
// each non-object column against its run by brute force (lane = column,
// ascending k: keep_old updates on <, take_new on <=, exact_edt.cpp:205/:275),
// and writes D, sqrt(D), labels and nearest columns with coalesced stores.
// This is the object->background polarity of C2 (94% object pixels, runs =
// disc chords) and of C1.
//
// A row with a run longer than kDenseRun is left to the merge-tree kernel
// (k_rows.cu, row-list mode): its index goes to `rest`.  Outputs the dense
// kernel already wrote for such a row are rewritten by that pass.
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kDenseRun = 1024;    // longest run allowed (the search per column stops at sqrt(D))
constexpr int kDenseWarps = 4;     // rows (warps) per CTA
constexpr int kDenseMaxW = 8192;

// per-warp shared memory: the staged row (wp halfwords) + its zero mask, 16 B aligned
__host__ __device__ __forceinline__ int dense_warp_bytes(int W) {
    const int wp = (W + 63) & ~63;
    return wp * 2 + (((wp / 32) * 4 + 15) & ~15);
}
inline int dense_smem_bytes(int W) { return kDenseWarps * dense_warp_bytes(W); }

template <bool TAKE_NEW>
__global__ void __launch_bounds__(32 * kDenseWarps) k_rows_dense(RowArgs a) {
    extern __shared__ uint4 dsm[];
    const int W = a.W;
    const int wp = (W + 63) & ~63;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint16_t* nrs = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(dsm) + warp * dense_warp_bytes(W));
    uint32_t* zmask = reinterpret_cast<uint32_t*>(nrs + wp);  // bit = column with g == 0
    const int nwords = (W + 31) >> 5;

    for (int64_t row = (int64_t)blockIdx.x * kDenseWarps + warp; row < a.total_rows;
         row += (int64_t)gridDim.x * kDenseWarps) {
        const int img = (int)(row / a.H);
        const uint32_t i = (uint32_t)(row - (int64_t)img * a.H);
        const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;
        const uint16_t* rowp = a.nr + img * a.nr_img_stride + (int64_t)i * a.Wp;
        // plane gate: fewer than half object pixels -> no short-run rows worth the staging
        // (row_done is zeroed by the caller); not a dense plane: jump to this
        // warp's first row of the next dense plane (32 plane counts per probe)
        if (a.plane_counts && (2 * a.plane_counts[img] < (unsigned long long)a.H * (unsigned long long)W ||
                               pts_plane(a.plane_counts, img, a.pts_gate))) {
            const int64_t nplanes = a.total_rows / a.H, stride = (int64_t)gridDim.x * kDenseWarps;
            int64_t next = nplanes;
            for (int64_t p0 = img + 1; p0 < nplanes; p0 += 32) {
                const int64_t p = p0 + lane;
                const bool dense = p < nplanes && 2 * a.plane_counts[p] >= (unsigned long long)a.H * (unsigned long long)W &&
                                   !pts_plane(a.plane_counts, (int)p, a.pts_gate);
                const unsigned m = __ballot_sync(0xffffffffu, dense);
                if (m) {
                    next = p0 + __ffs(m) - 1;
                    break;
                }
            }
            const int64_t first = next * a.H;  // rows >= first with row == start (mod stride)
            row += ((first - row + stride - 1) / stride - 1) * stride;  // the loop step reaches it
            continue;
        }

        // ---- stage the row (16-byte loads, all in flight) and its zero mask ----
        if (a.vec_nr) {
            const uint4* src = reinterpret_cast<const uint4*>(rowp);
            uint4* dst = reinterpret_cast<uint4*>(nrs);
            const int nvec = (W + 7) >> 3;
#pragma unroll 4
            for (int v = lane; v < nvec; v += 32) dst[v] = __ldg(src + v);
        } else {
            for (int j = lane; j < W; j += 32) {
                const int t = a.tile_cols >= W ? 0 : j / a.tile_cols;
                nrs[j] = __ldg(rowp + t * a.tile_stride + (j - t * a.tile_cols));
            }
        }
        __syncwarp();
        for (int w = lane; w < nwords; w += 32) {  // lane builds whole words: 4 x 16 B reads
            const uint4* q = reinterpret_cast<const uint4*>(nrs + 32 * w);
            uint32_t z = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint4 v = q[u];
                const uint32_t h[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int b = 8 * u + 2 * t;
                    z |= (uint32_t)((h[t] & 0xffffu) == gi && 32 * w + b < W) << b;
                    z |= (uint32_t)((h[t] >> 16) == gi && 32 * w + b + 1 < W) << (b + 1);
                }
            }
            zmask[w] = z;
        }
        __syncwarp();

        // ---- longest run of non-zero columns (row ends bound runs too) ----
        // lane w-slice: runs inside words are found from the word boundaries' view
        bool sparse = false;
        {
            int last = -1;  // last zero column seen
            for (int w = 0; w < nwords && !sparse; w += 32) {
                const int myw = w + lane;
                const uint32_t m = myw < nwords ? zmask[myw] : 0u;
                // zero columns inside my word: first / last, and the longest inner run
                int first = -1, lastz = -1, inner = 0;
                if (m) {
                    first = 32 * myw + __ffs(m) - 1;
                    lastz = 32 * myw + 31 - __clz(m);
                    uint32_t mm = m;  // inner runs: gaps between consecutive set bits
                    int prev = -1;
                    while (mm) {
                        const int b = __ffs(mm) - 1;
                        if (prev >= 0) inner = max(inner, b - prev - 1);
                        prev = b;
                        mm &= mm - 1;
                    }
                }
                // carry the last zero column across words in order (inclusive max-scan)
                int lz = lastz;
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, lz, o);
                    if (lane >= o) lz = max(lz, v);
                }
                int before = __shfl_up_sync(0xffffffffu, lz, 1);
                if (lane == 0) before = -1;
                before = max(before, last);
                // run ending at my first zero, and the run after the row's last zero
                int run = inner;
                if (first >= 0) run = max(run, first - before - 1);
                const int lastall = __shfl_sync(0xffffffffu, lz, 31);
                last = max(last, lastall);
                if (w + 32 >= nwords) run = max(run, W - 1 - last);  // trailing run
                sparse = __any_sync(0xffffffffu, run > kDenseRun);
            }
        }
        if (lane == 0) a.row_done[row] = sparse ? 0 : 1;
        if (sparse) {
            __syncwarp();
            continue;
        }

        int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + img * a.sD) + (int64_t)i * W : nullptr;
        float* Srow = a.S ? reinterpret_cast<float*>(a.S + img * a.sS) + (int64_t)i * W : nullptr;
        int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + img * a.sL) + (int64_t)i * W : nullptr;
        int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + img * a.sN) + (int64_t)i * W : nullptr;

        // ---- every column: outward search from j.  h^2 > best ends it (a later
        // candidate is farther); an object column stops at h = 0, the others
        // within their run (<= kDenseRun + 1).  Ties: smaller column for
        // keep_old, larger for take_new, explicitly (the visiting order
        // alternates sides). ----
        for (int w = 0; w < nwords; ++w) {
            const int j = 32 * w + lane;
            if (j >= W) break;
            if (zmask[w] == 0xffffffffu) {  // 32 object pixels: D = 0, own column (warp-uniform)
                if (Drow) __stcs(Drow + j, 0);
                if (Srow) __stcs(Srow + j, 0.0f);
                if (Lrow) __stcs(Lrow + j, (int32_t)(gi * (uint32_t)W + (uint32_t)j));
                if (Nrow) __stcs(Nrow + j, j);
                continue;
            }
            uint32_t best = kInfU, bk = 0, br = kNoRow;
            const int hmax = max(j, W - 1 - j);
            for (int h = 0; h <= hmax && (uint32_t)(h * h) <= best; ++h) {
                const uint32_t hh = (uint32_t)(h * h);
                // left j-h: the smallest column seen so far (wins keep_old ties);
                // right j+h: the largest (wins take_new ties); off-row -> none
                const int kl = j - h, kr = j + h;
                const uint32_t rl = kl >= 0 ? nrs[kl] : kNoRow;
                const uint32_t rr = (h > 0 && kr < W) ? nrs[kr] : kNoRow;
                if (rl != kNoRow) {
                    const uint32_t av = gi > rl ? gi - rl : rl - gi;
                    const uint32_t d = av * av + hh;
                    if (TAKE_NEW ? d < best : d <= best) { best = d; bk = (uint32_t)kl; br = rl; }
                }
                if (rr != kNoRow) {
                    const uint32_t av = gi > rr ? gi - rr : rr - gi;
                    const uint32_t d = av * av + hh;
                    if (TAKE_NEW ? d <= best : d < best) { best = d; bk = (uint32_t)kr; br = rr; }
                }
            }
            const bool inf = best == kInfU;
            if (Drow) __stcs(Drow + j, inf ? DFC_INF_I32 : (int32_t)best);
            if (Srow) __stcs(Srow + j, dist_f32(best));
            if (Lrow) __stcs(Lrow + j, inf ? -1 : (int32_t)(br * (uint32_t)W + bk));
            if (Nrow) __stcs(Nrow + j, inf ? -1 : (int32_t)bk);
        }
        __syncwarp();
    }
}

template <bool TAKE_NEW>
inline const void* dense_kernel_ptr() {
    return (const void*)k_rows_dense<TAKE_NEW>;
}

}  // namespace dfc
