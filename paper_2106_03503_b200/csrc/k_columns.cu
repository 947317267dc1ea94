// k_columns.cu -- stage 1 of the separable EDT: the per-column nearest-object scan.
//
// Replaces vertical_pass = init_distance_map + vertical_down_pass +
// vertical_up_pass (exact_edt.cpp:74-117, grid.cpp:85-91) and the src_row
// bookkeeping of voronoi_labels (exact_edt.cpp:327-360).  Instead of walking
// each column serially through a uint64 map (stride cols*8 B), the image is
// cut into bands of 32 rows; a thread owns 4 adjacent columns of one band and
// turns the band into four 32-bit row masks with ONE coalesced 4-byte load
// per row.  Nearest object above/below inside the band is then a clz/ffs on
// the mask; across bands it comes from per-(band, column) carries:
//
//   K1a k_band_summary : first/last object row of every (band, column)
//   K1b k_band_scan    : per column, turns them into "nearest object row
//                        above this band" / "below this band" carries
//   K1c k_band_fill    : per pixel, the nearest object row in its column
//                        (uint16, upper row on ties -- the reference's strict
//                        '>' keeps the down-pass feature, exact_edt.cpp:351),
//                        or the squared vertical distance itself (int32).
//
// Both polarities (object = nonzero, and object = zero for the inverted image,
// grid.cpp:38-44) come out of one read of the input ("slots").
#include "dfc_kernels.cuh"

namespace dfc {

// Load the 32 rows of one band for 4 columns [j0, j0+4) and return one row
// mask per column (bit r = row r0+r is an object pixel, i.e. nonzero byte).
__device__ __forceinline__ void band_masks(const uint8_t* __restrict__ base, int64_t pitch,
                                           int nrows, int j0, int W, bool vec,
                                           uint32_t (&m)[4]) {
    m[0] = m[1] = m[2] = m[3] = 0u;
    if (vec && j0 + 3 < W) {
        uint32_t v[kBand];
        const uint8_t* p = base + j0;
#pragma unroll
        for (int r = 0; r < kBand; ++r, p += pitch)
            v[r] = r < nrows ? __ldg(reinterpret_cast<const uint32_t*>(p)) : 0u;
        // sparse images: most threads see 128 zero bytes (16 three-input ORs)
        uint32_t any = 0u;
#pragma unroll
        for (int r = 0; r < kBand; r += 2) any |= v[r] | v[r + 1];
        if (any == 0u) return;
        // 4 x 32 bit transpose: x[g] byte c bit b = row 8g + b of column c
        // (one 0xff-per-nonzero-byte compare and one masked OR per row), then
        // each column's word gathers byte c of x[0..3] with three byte permutes
        uint32_t x[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int r = 0; r < kBand; ++r) x[r >> 3] |= __vcmpne4(v[r], 0u) & (0x01010101u << (r & 7));
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t sel = (uint32_t)c | ((uint32_t)(c + 4) << 4);
            m[c] = __byte_perm(__byte_perm(x[0], x[1], sel), __byte_perm(x[2], x[3], sel), 0x5410);
        }
    } else {
        for (int r = 0; r < nrows; ++r) {
            const uint8_t* row = base + r * pitch;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (j0 + c < W && row[j0 + c] != 0) m[c] |= 1u << r;
        }
    }
}



// K1a: grid (ceil(W/4)/blockDim, nb, n_img)
// counts (nullable): object pixels per plane [slot][img], accumulated with one
// atomic per warp (the row pass's dense-plane gate, k_rows_dense.cu).
__global__ void k_band_summary(ColArgs a, uint16_t* __restrict__ first, uint16_t* __restrict__ last,
                               unsigned long long* __restrict__ counts) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int j0 = 4 * g;
    const bool live = j0 < a.W;  // no early exit: the count reduction needs the whole warp
    const int b = blockIdx.y, im = blockIdx.z;
    const int r0 = b * kBand;
    const int nrows = min(kBand, a.H - r0);
    const uint32_t valid = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    if (live) band_masks(a.img + im * a.img_stride + (int64_t)r0 * a.pitch, a.pitch, nrows, j0, a.W, a.vec, m);
    if (a.bmask && live)
        *reinterpret_cast<uint4*>(a.bmask + ((int64_t)im * a.nb + b) * a.Wp + j0) = make_uint4(m[0], m[1], m[2], m[3]);
    // a warp whose 128 columns x 32 rows hold no nonzero byte (most warps of a
    // sparse image), object = nonzero only: no object row, no count, no point
    if (a.npol == 1 && a.pol0 == 0 && !__any_sync(0xffffffffu, (m[0] | m[1] | m[2] | m[3]) != 0u)) {
        if (!live) return;
        const int64_t off = ((int64_t)im * a.nb + b) * a.Wp + j0;
        const uint32_t none2 = (uint32_t)kNoRow | ((uint32_t)kNoRow << 16);
        *reinterpret_cast<uint2*>(first + off) = make_uint2(none2, none2);
        *reinterpret_cast<uint2*>(last + off) = make_uint2(none2, none2);
        if (a.objcol && (threadIdx.x & 7) == 0) {
            const int Ww = (a.W + 31) >> 5;
            if ((j0 >> 5) < Ww) a.objcol[((int64_t)im * a.nb + b) * Ww + (j0 >> 5)] = 0u;
        }
        return;
    }
    for (int s = 0; s < a.npol; ++s) {
        const int pol = a.pol0 + s;
        uint16_t f[4], l[4];
        uint32_t mk[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            mk[c] = (live && j0 + c < a.W) ? pol_mask(m[c], pol, valid) : 0u;
            f[c] = mk[c] ? (uint16_t)(r0 + __ffs(mk[c]) - 1) : kNoRow;
            l[c] = mk[c] ? (uint16_t)(r0 + 31 - __clz(mk[c])) : kNoRow;
        }
        if (a.objcol) {  // 4 bits per thread, 8 threads per 32-column word
            const int lane = threadIdx.x & 31;
            uint32_t v = ((uint32_t)(mk[0] != 0u) | ((uint32_t)(mk[1] != 0u) << 1) | ((uint32_t)(mk[2] != 0u) << 2) |
                          ((uint32_t)(mk[3] != 0u) << 3)) << (4 * (lane & 7));
            v |= __shfl_xor_sync(0xffffffffu, v, 1);
            v |= __shfl_xor_sync(0xffffffffu, v, 2);
            v |= __shfl_xor_sync(0xffffffffu, v, 4);
            const int Ww = (a.W + 31) >> 5;
            if ((lane & 7) == 0 && (j0 >> 5) < Ww)
                a.objcol[(((int64_t)s * a.n_img + im) * a.nb + b) * Ww + (j0 >> 5)] = v;
        }
        if (counts) {
            const unsigned mine = (unsigned)(__popc(mk[0]) + __popc(mk[1]) + __popc(mk[2]) + __popc(mk[3]));
            const unsigned long long c = __reduce_add_sync(0xffffffffu, mine);  // <= 32 x 128: one REDUX
            const int lane = threadIdx.x & 31;
            const int64_t plane = (int64_t)s * a.n_img + im;
            unsigned long long old = 0;
            if (lane == 0 && c) old = atomicAdd(counts + plane, c);
            old = __shfl_sync(0xffffffffu, old, 0);
            // the plane's first kPtsCap object pixels go to its point list (the
            // running count is the position; a longer plane's list is unused)
            if (a.pts && c && old + c <= (unsigned long long)kPtsCap) {
                unsigned pre = mine;  // inclusive prefix of the per-lane counts
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned v = __shfl_up_sync(0xffffffffu, pre, o);
                    if (lane >= o) pre += v;
                }
                uint32_t* dst = a.pts + plane * kPtsCap + old + (pre - mine);
                for (int cc = 0; cc < 4; ++cc)
                    for (uint32_t m = mk[cc]; m; m &= m - 1)
                        *dst++ = ((uint32_t)(j0 + cc) << 16) | (uint32_t)(r0 + __ffs(m) - 1);
            }
        }
        if (!live) continue;
        const int64_t off = (((int64_t)s * a.n_img + im) * a.nb + b) * a.Wp + j0;
        *reinterpret_cast<uint2*>(first + off) =
            make_uint2(f[0] | ((uint32_t)f[1] << 16), f[2] | ((uint32_t)f[3] << 16));
        *reinterpret_cast<uint2*>(last + off) =
            make_uint2(l[0] | ((uint32_t)l[1] << 16), l[2] | ((uint32_t)l[3] << 16));
    }
}

// K1b (short columns, <= 64 bands): one thread per (column, plane), serial
// over the bands with 16 independent loads in flight; same in-place result as
// the chunked scan below.
__global__ void __launch_bounds__(256, 4) k_band_scan_serial(int W, int Wp, int nb, int64_t n_planes, uint16_t* __restrict__ first,
                                   uint16_t* __restrict__ last, const unsigned long long* skip_counts) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t plane = blockIdx.y;
    if (j >= W || plane >= n_planes) return;
    if (skip_counts && skip_counts[plane] <= (unsigned long long)kPtsCap) return;  // point plane
    uint16_t* F = first + plane * nb * (int64_t)Wp + j;
    uint16_t* Lp = last + plane * nb * (int64_t)Wp + j;
    // both scans at once, 8 bands of each loaded before any is used: the
    // exclusive prefix max of last (forward) and suffix min of first (backward)
    constexpr int kB = 8;
    uint16_t runL = kNoRow, runF = kNoRow;
    for (int b = 0; b < nb; b += kB) {
        uint16_t tl[kB], tf[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (b + u < nb) {
                tl[u] = Lp[(int64_t)(b + u) * Wp];
                tf[u] = F[(int64_t)(nb - 1 - b - u) * Wp];
            }
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (b + u < nb) {
                Lp[(int64_t)(b + u) * Wp] = runL;
                if (tl[u] != kNoRow) runL = tl[u];
                F[(int64_t)(nb - 1 - b - u) * Wp] = runF;
                if (tf[u] != kNoRow) runF = tf[u];
            }
    }
}

// K1b: per column, in place: last[b] becomes the nearest object row ABOVE band
// b (exclusive prefix-max over bands: rows grow with the band index, kNoRow =
// absent), first[b] the nearest object row BELOW it (exclusive suffix-min).
// CTA = 128 columns (4 per thread, 8-byte accesses) x nc band chunks (nc <=
// 32); a thread scans its chunk twice (aggregate, then carry-in + write) --
// coalesced across the columns, and parallel over the chunks instead of a
// serial walk over all bands.
__global__ void __launch_bounds__(1024) k_band_scan(int W, int Wp, int nb, int64_t n_planes,
                                                    uint16_t* __restrict__ first, uint16_t* __restrict__ last,
                                                    const unsigned long long* skip_counts) {
    if (skip_counts && blockIdx.y < n_planes && skip_counts[blockIdx.y] <= (unsigned long long)kPtsCap)
        return;  // point plane (CTA-uniform)
    __shared__ int agg_last[32][129];
    __shared__ int agg_first[32][129];
    const int cx = threadIdx.x & 31, ch = threadIdx.x >> 5, nc = blockDim.x >> 5;
    const int j0 = blockIdx.x * 128 + 4 * cx;  // Wp % 8 == 0: the 4 columns are in the row
    const int64_t plane = blockIdx.y;
    const int per = (nb + nc - 1) / nc;
    const int b0 = ch * per, b1 = min(b0 + per, nb);
    uint2* F = reinterpret_cast<uint2*>(first + plane * nb * (int64_t)Wp + j0);
    uint2* Lp = reinterpret_cast<uint2*>(last + plane * nb * (int64_t)Wp + j0);
    const int64_t step = Wp / 4;  // uint2 per row of bands
    const bool ok = j0 < W && plane < n_planes;
    auto split = [](uint2 v, int (&o)[4]) {
        o[0] = (int)(v.x & 0xffffu); o[1] = (int)(v.x >> 16); o[2] = (int)(v.y & 0xffffu); o[3] = (int)(v.y >> 16);
    };
    // every pass loads kB bands before using any (independent loads in flight
    // instead of one load latency per band)
    constexpr int kB = 8;
    int mx[4] = {-1, -1, -1, -1}, mn[4] = {0x10000, 0x10000, 0x10000, 0x10000};
    if (ok)
        for (int bb = b0; bb < b1; bb += kB) {
            uint2 lv[kB], fv[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u)
                if (bb + u < b1) {
                    lv[u] = Lp[(int64_t)(bb + u) * step];
                    fv[u] = F[(int64_t)(bb + u) * step];
                }
#pragma unroll
            for (int u = 0; u < kB; ++u)
                if (bb + u < b1) {
                    int l[4], f[4];
                    split(lv[u], l);
                    split(fv[u], f);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (l[t] != kNoRow) mx[t] = l[t];                   // rows increase with b: latest = max
                        if (f[t] != kNoRow && mn[t] == 0x10000) mn[t] = f[t];  // earliest in the chunk = min
                    }
                }
        }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        agg_last[ch][4 * cx + t] = mx[t];
        agg_first[ch][4 * cx + t] = mn[t];
    }
    __syncthreads();
    // carries into each chunk: exclusive prefix max / suffix min over the nc
    // chunk aggregates of every column, by warp scans (lane = chunk; warp w
    // handles columns w, w + nc, ...), written back in place
    for (int col = ch; col < 128; col += nc) {
        const int c = cx;
        int vl = c < nc ? agg_last[c][col] : -1;
        int vf = c < nc ? agg_first[c][col] : 0x10000;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ul = __shfl_up_sync(0xffffffffu, vl, o), df = __shfl_down_sync(0xffffffffu, vf, o);
            if (c >= o) vl = max(vl, ul);
            if (c + o < 32) vf = min(vf, df);
        }
        // inclusive -> exclusive
        int el = __shfl_up_sync(0xffffffffu, vl, 1), ef = __shfl_down_sync(0xffffffffu, vf, 1);
        if (c == 0) el = -1;
        if (c + 1 >= nc) ef = 0x10000;
        __syncwarp();
        if (c < nc) {
            agg_last[c][col] = el;
            agg_first[c][col] = ef;
        }
    }
    __syncthreads();
    if (!ok) return;
    int above[4], below[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        above[t] = agg_last[ch][4 * cx + t];
        below[t] = agg_first[ch][4 * cx + t];
    }
    auto pack = [](const int (&v)[4], int none) -> uint2 {
        uint32_t w[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) w[t] = v[t] == none ? kNoRow : (uint32_t)v[t];
        return make_uint2(w[0] | (w[1] << 16), w[2] | (w[3] << 16));
    };
    for (int bb = b0; bb < b1; bb += kB) {  // exclusive prefix max
        uint2 lv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (bb + u < b1) lv[u] = Lp[(int64_t)(bb + u) * step];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (bb + u < b1) {
                int l[4];
                split(lv[u], l);
                Lp[(int64_t)(bb + u) * step] = pack(above, -1);
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (l[t] != kNoRow) above[t] = l[t];
            }
    }
    for (int bb = b1 - 1; bb >= b0; bb -= kB) {  // exclusive suffix min
        uint2 fv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (bb - u >= b0) fv[u] = F[(int64_t)(bb - u) * step];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (bb - u >= b0) {
                int f[4];
                split(fv[u], f);
                F[(int64_t)(bb - u) * step] = pack(below, 0x10000);
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (f[t] != kNoRow) below[t] = f[t];
            }
    }
}

// K1c: per pixel nearest object row (OUT_SQ=false: uint16 plane [slot][img][H][Wp])
// or the squared vertical distance (OUT_SQ=true: int32, dense [img][H][W]).
constexpr int kFillBands = 8;

template <bool OUT_SQ>
__global__ void __launch_bounds__(128, 8) k_band_fill(ColArgs a, const uint16_t* __restrict__ below,
                            const uint16_t* __restrict__ above, uint16_t* __restrict__ nr,
                            int32_t* __restrict__ vsq) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int j0 = 4 * g;
    if (j0 >= a.W) return;
    const int im = blockIdx.z;
    // planes without a nearest-row plane: point planes (k_rows_pts) and, with
    // skip_full, planes k_rows_anc stages from the bands (CTA-uniform)
    auto skip_plane = [&](int s) {
        const int64_t p = (int64_t)s * a.n_img + im;
        if (a.pts && a.pcounts[p] <= (unsigned long long)kPtsCap) return true;
        if (!a.pcounts) return false;
        const bool sparse = lr_plane(a.pcounts, (int)p, a.H, a.W);
        return sparse ? a.skip_sparse : a.skip_full;
    };
    if (a.pts || a.skip_full || a.skip_sparse) {
        bool all = true;
        for (int s = 0; s < a.npol; ++s) all = all && skip_plane(s);
        if (all) return;
    }
    // several bands per CTA for batches (a skipped plane costs few CTAs), one
    // for single images (loads of consecutive bands overlap across CTAs)
    const int bpc = (a.nb + (int)gridDim.y - 1) / (int)gridDim.y;
    for (int b = blockIdx.y * bpc; b < min(a.nb, (int)(blockIdx.y + 1) * bpc); ++b) {
    const int r0 = b * kBand;
    const int nrows = min(kBand, a.H - r0);
    const uint32_t valid = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
    uint32_t m[4];
    if (a.bmask) {  // K1a's masks: 16 bytes instead of 32 image rows
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(a.bmask + ((int64_t)im * a.nb + b) * a.Wp + j0));
        m[0] = q.x; m[1] = q.y; m[2] = q.z; m[3] = q.w;
    } else {
        band_masks(a.img + im * a.img_stride + (int64_t)r0 * a.pitch, a.pitch, nrows, j0, a.W, a.vec, m);
    }
    for (int s = 0; s < a.npol; ++s) {
        const int pol = a.pol0 + s;
        if ((a.pts || a.skip_full || a.skip_sparse) && skip_plane(s)) continue;
        const int64_t coff = (((int64_t)s * a.n_img + im) * a.nb + b) * a.Wp + j0;
        const uint2 ab = *reinterpret_cast<const uint2*>(above + coff);
        const uint2 bl = *reinterpret_cast<const uint2*>(below + coff);
        const uint32_t ca[4] = {ab.x & 0xffffu, ab.x >> 16, ab.y & 0xffffu, ab.y >> 16};
        const uint32_t cb[4] = {bl.x & 0xffffu, bl.x >> 16, bl.y & 0xffffu, bl.y >> 16};
        uint32_t mk[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) mk[c] = pol_mask(m[c], pol, valid);
        auto row_out = [&](int r) {
            const uint32_t i = r0 + r;
            uint32_t out[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t up = mk[c] & (0xffffffffu >> (31 - r));   // rows r0..i
                const uint32_t dn = mk[c] >> r;                          // rows i..
                const uint32_t ra = up ? (uint32_t)(r0 + 31 - __clz(up)) : ca[c];
                const uint32_t rb = dn ? (uint32_t)(i + __ffs(dn) - 1) : cb[c];
                out[c] = pick_nearest(i, ra, rb);
            }
            if (!OUT_SQ) {
                const int64_t off = (((int64_t)s * a.n_img + im) * a.H + i) * a.Wp + j0;
                *reinterpret_cast<uint2*>(nr + off) =
                    make_uint2(out[0] | (out[1] << 16), out[2] | (out[3] << 16));
            } else {
                int32_t* row = vsq + (((int64_t)s * a.n_img + im) * a.H + i) * (int64_t)a.W;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (j0 + c >= a.W) break;
                    const uint32_t r_ = out[c];
                    const uint32_t d = r_ == kNoRow ? (uint32_t)DFC_INF_I32
                                                    : sq(i > r_ ? i - r_ : r_ - i);
                    row[j0 + c] = (int32_t)d;
                }
            }
        };
        if (!OUT_SQ && (mk[0] | mk[1] | mk[2] | mk[3]) == 0) {
            // no object of this polarity in the band's 4 columns (sparse images):
            // rows up to (ca + cb) / 2 take the carry above (the upper row on a
            // tie), the others the carry below
            int thr[4];
#pragma unroll
            for (int c = 0; c < 4; ++c)
                thr[c] = ca[c] == kNoRow ? -1 : (cb[c] == kNoRow ? 0x7fffffff : (int)((ca[c] + cb[c]) >> 1));
            const uint32_t lo0 = ca[0] | (ca[1] << 16), lo1 = ca[2] | (ca[3] << 16);
            const uint32_t hi0 = cb[0] | (cb[1] << 16), hi1 = cb[2] | (cb[3] << 16);
            uint2* dst = reinterpret_cast<uint2*>(nr + (((int64_t)s * a.n_img + im) * a.H + r0) * a.Wp + j0);
            const int rstep = a.Wp >> 2;  // uint2 per row
#pragma unroll 4
            for (int r = 0; r < nrows; ++r, dst += rstep) {
                const int i = r0 + r;
                const uint32_t x0 = i <= thr[0] ? (lo0 & 0xffffu) : (hi0 & 0xffffu);
                const uint32_t x1 = i <= thr[1] ? (lo0 & 0xffff0000u) : (hi0 & 0xffff0000u);
                const uint32_t x2 = i <= thr[2] ? (lo1 & 0xffffu) : (hi1 & 0xffffu);
                const uint32_t x3 = i <= thr[3] ? (lo1 & 0xffff0000u) : (hi1 & 0xffff0000u);
                *dst = make_uint2(x0 | x1, x2 | x3);
            }
            continue;
        }
        if (nrows == kBand) {  // full band: fully unrolled (masks, shifts constant-folded)
#pragma unroll
            for (int r = 0; r < kBand; ++r) row_out(r);
        } else {
            for (int r = 0; r < nrows; ++r) row_out(r);
        }
    }
    }  // bands
}

// Per-direction vertical passes over an arbitrary squared-distance map
// (uint64, in place, INF = UINT64_MAX): vertical_down_pass / vertical_up_pass
// (exact_edt.cpp:74-110) -- the odd-step increment chain with the strict '>'
// update and the step reset, same unsigned arithmetic.  One thread per
// column (coalesced across the warp), serial over rows, 4 rows of loads in
// flight ahead of the dependent chain.
template <bool UP>
__global__ void k_vpass_u64(uint64_t* __restrict__ dm, int64_t rows, int64_t cols, int64_t pitch) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols || rows < 2) return;
    constexpr uint64_t kInf = ~0ull;
    uint64_t* col = dm + j;
    const int64_t step_i = UP ? -pitch : pitch;
    uint64_t* p = col + (UP ? (rows - 1) * pitch : 0);
    uint64_t prev = *p;  // row 0 (down) / rows-1 (up) is never updated
    uint64_t step = 1;
    int64_t n = rows - 1;
    p += step_i;
    while (n > 0) {
        const int c = n >= 4 ? 4 : (int)n;
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = u < c ? p[u * step_i] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (u >= c) break;
            uint64_t cur = v[u];
            if (prev != kInf && (cur == kInf || cur > prev + step)) {
                cur = prev + step;
                p[u * step_i] = cur;
                step += 2;
            } else {
                step = 1;
            }
            prev = cur;
        }
        p += c * step_i;
        n -= c;
    }
}

template __global__ void k_band_fill<false>(ColArgs, const uint16_t*, const uint16_t*, uint16_t*, int32_t*);
template __global__ void k_band_fill<true>(ColArgs, const uint16_t*, const uint16_t*, uint16_t*, int32_t*);

}  // namespace dfc
