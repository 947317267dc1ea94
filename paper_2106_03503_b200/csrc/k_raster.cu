// k_raster.cu -- the approximate transforms of config 4 from the stage-1 output.
//
// Replaces the reference's sequential two-pass raster scans
// cityblock_sequential (propagation.cpp:16-34, 90-95) and chamfer34
// (propagation.cpp:60-88, 104-109), plus a chessboard transform (the
// reference only has the brute-force test oracle, proj/tests/oracles.hpp:52-55).
// The raster dependency (every cell waits for its upper-left neighbours) is
// not needed for the final maps: with a_k = vertical pixel distance to the
// nearest object in column k (stage 1, k_columns.cu),
//     city-block  = min_k  a_k + |j-k|
//     chessboard  = min_k  max(a_k, |j-k|)
//     chamfer-3-4 = min_k  3*max(a_k,|j-k|) + min(a_k,|j-k|)
// (SURVEY.md finding 6; re-verified in tests/test_oracle.py::
// test_separable_closed_forms against the reference's own raster results).
// One CTA per row: city-block by two min-plus scans (thread-local segment
// scans + a CTA-wide prefix/suffix min for the segment carries), chessboard
// and chamfer by an outward window search per cell that stops as soon as the
// horizontal offset alone can no longer improve (the reference's own early
// exit rule, exact_edt.cpp:161-180).
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kBig = 0x1fffffff;  // "no object in this column"; 4 * kBig still fits int32


// padded index: one pad word per L-column segment (segment-strided and
// column-contiguous accesses are both bank-conflict free); L = 2^lg
__device__ __forceinline__ int pidx(int j, int lg) { return j + (j >> lg); }

__global__ void __launch_bounds__(1024) k_raster(RasterArgs a) {
    extern __shared__ int rs[];
    const int T = a.T, L = a.L, W = a.W;
    const int lg = 31 - __clz(L);
    const int s = threadIdx.x;
    const int i = blockIdx.x;
    const int padW = W + W / L + 1;
    int* av = rs + 2;           // [-2, padW) vertical distance a_k (kBig = none); pidx(-1), pidx(W): kBig
    int* l1 = av + padW;        // [padW] city-block row
    int* v = l1 + padW;         // [T] scan scratch
    int* w = v + T;             // [T]

    const uint16_t* src = a.nr + (int64_t)i * a.Wp;
    int any = 0;
    for (int j = s; j < W; j += T) {
        const uint32_t r = src[j];
        const int d = r == kNoRow ? kBig : (int)(i > (int)r ? i - (int)r : (int)r - i);
        av[pidx(j, lg)] = d;
        any |= d < kBig;
    }
    if (s == 0) {
        av[pidx(-1, lg)] = kBig;
        av[pidx(W, lg)] = kBig;
    }
    const bool row_has = __syncthreads_or(any);
    int32_t* crow = a.city ? a.city + (int64_t)i * W : nullptr;
    int32_t* brow = a.chess ? a.chess + (int64_t)i * W : nullptr;
    int32_t* mrow = a.cham ? a.cham + (int64_t)i * W : nullptr;
    if (!row_has) {  // featureless image: all infinite (test_propagation.cpp:73-78)
        for (int j = s; j < W; j += T) {
            if (crow) crow[j] = DFC_INF_I32;
            if (brow) brow[j] = DFC_INF_I32;
            if (mrow) mrow[j] = DFC_INF_I32;
        }
        return;
    }

    // ---- city-block: local forward/backward min-plus scans per segment ----
    const int c0 = s * L, c1 = min(c0 + L, W);
    int fend = kBig, bbeg = kBig;
    {
        int f = kBig;
        for (int j = c0; j < c1; ++j) f = min(av[pidx(j, lg)], f + 1);
        fend = f;
        int b = kBig;
        for (int j = c1 - 1; j >= c0; --j) b = min(av[pidx(j, lg)], b + 1);
        bbeg = b;
    }
    // carries: fwd(c0-1) = min_{s'<s} (fend_s' - (s'+1)L) + sL
    //          bwd(c1)   = min_{s'>s} (bbeg_s' + s'L) - (s+1)L
    v[s] = fend - (s + 1) * L;
    w[s] = bbeg + s * L;
    __syncthreads();
    for (int off = 1; off < T; off <<= 1) {  // Hillis-Steele inclusive prefix/suffix min
        const int pv = s >= off ? v[s - off] : kBig;
        const int pw = s + off < T ? w[s + off] : kBig;
        __syncthreads();
        v[s] = min(v[s], pv);
        w[s] = min(w[s], pw);
        __syncthreads();
    }
    if (c0 < W) {
        int f = s > 0 ? min(kBig, v[s - 1] + s * L) : kBig;   // fwd(c0 - 1)
        for (int j = c0; j < c1; ++j) {
            f = min(av[pidx(j, lg)], f + 1);
            l1[pidx(j, lg)] = f;
        }
        int b = s + 1 < T ? min(kBig, w[s + 1] - (s + 1) * L) : kBig;  // bwd(c1)
        for (int j = c1 - 1; j >= c0; --j) {
            b = min(av[pidx(j, lg)], b + 1);
            l1[pidx(j, lg)] = min(l1[pidx(j, lg)], b);
        }
    }
    __syncthreads();

    // ---- chessboard / chamfer-3-4: outward window search per cell ----
    // bch >= 3 * binf throughout, so 3h >= bch ends both searches; columns
    // outside the row read the kBig sentinels at pidx(-1) and pidx(W).
    for (int j = s; j < W; j += T) {
        const int aj = av[pidx(j, lg)];
        int binf = aj, bch = 3 * aj;
        const int hmax = max(j, W - 1 - j);
        for (int h = 1; 3 * h < bch && h <= hmax; ++h) {
            const int al = av[pidx(max(j - h, -1), lg)];
            const int ar = av[pidx(min(j + h, W), lg)];
            const int ml = max(al, h), mr = max(ar, h);
            binf = min(binf, min(ml, mr));
            bch = min(bch, min(3 * ml + min(al, h), 3 * mr + min(ar, h)));
        }
        if (crow) __stcs(crow + j, l1[pidx(j, lg)]);
        if (brow) __stcs(brow + j, binf);
        if (mrow) __stcs(mrow + j, bch);
    }
}

// ---- float distances from a squared map (the row pass's epilogue, standalone) ----
__global__ void k_sqrt_i32(const int32_t* __restrict__ d, float* __restrict__ out, int64_t n) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        out[p] = dist_f32((uint32_t)d[p]);
}

// ---- label ordinals (LabelMap ids, grid.cpp:29-36) ----
// K4a: one warp per row: per-32-column word object masks and in-row prefix counts.
__global__ void k_ord_rows(const uint8_t* __restrict__ img, int64_t pitch, int H, int W, int nw,
                           uint32_t* __restrict__ masks, uint32_t* __restrict__ wpre,
                           uint32_t* __restrict__ rowcnt) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= H) return;
    const uint8_t* row = img + (int64_t)warp * pitch;
    uint32_t run = 0;
    for (int wd = 0; wd < nw; ++wd) {
        const int j = wd * 32 + lane;
        const uint32_t m = __ballot_sync(0xffffffffu, j < W && row[j] != 0);
        if (lane == 0) {
            masks[(int64_t)warp * nw + wd] = m;
            wpre[(int64_t)warp * nw + wd] = run;
        }
        run += __popc(m);
    }
    if (lane == 0) rowcnt[warp] = run;
}

// K4b: exclusive scan of the per-row counts (single CTA, 1024 threads).
__global__ void k_ord_scan(const uint32_t* __restrict__ rowcnt, uint32_t* __restrict__ rowbase, int H) {
    __shared__ uint32_t part[1024];
    const int t = threadIdx.x;
    const int per = (H + 1023) / 1024;
    const int b0 = t * per, b1 = min(b0 + per, H);
    uint32_t sum = 0;
    for (int r = b0; r < b1; ++r) sum += rowcnt[r];
    part[t] = sum;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t pv = t >= off ? part[t - off] : 0u;
        __syncthreads();
        part[t] += pv;
        __syncthreads();
    }
    uint32_t run = t > 0 ? part[t - 1] : 0u;
    for (int r = b0; r < b1; ++r) {
        rowbase[r] = run;
        run += rowcnt[r];
    }
}

// K4c: ordinal of the labelled pixel.
__global__ void k_ord_map(const int32_t* __restrict__ label, int64_t n, int W, int nw,
                          const uint32_t* __restrict__ masks, const uint32_t* __restrict__ wpre,
                          const uint32_t* __restrict__ rowbase, uint32_t* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t lb = label[p];
        uint32_t o = 0xffffffffu;
        if (lb >= 0) {
            const int r = lb / W, c = lb - r * W;
            const int64_t wi = (int64_t)r * nw + (c >> 5);
            o = rowbase[r] + wpre[wi] + __popc(masks[wi] & ((1u << (c & 31)) - 1u));
        }
        out[p] = o;
    }
}

}  // namespace dfc
