// k_rows_lr.cu -- stage 2 as a LANE-PER-ROW chunk scan with entry-level
// eager finalisation, then a warp-cooperative fill.
//
// Same result as k_rows.cu (envelope_rows / meijster_scan / voronoi label
// assembly, exact_edt.cpp:190-283, :362-369), different decomposition.  A warp
// owns 32 consecutive rows and one column chunk [c0, c1); every lane runs the
// reference's stack algorithm (exact_edt.cpp:208-223) over ITS row, left to
// right (one 16-byte load = 8 columns, prefetched one group ahead).  There is
// no merge step: the chunks of a row are independent.
//
//  bounds    owners are monotone in j (smallest and largest minimiser alike),
//            so every owner of [c0, c1) lies in [owner(c0-1), owner(c1-1)]:
//            each lane finds those two owners exactly (outward search from the
//            column until the next unexamined distance d has d^2 > best) and
//            scans only that range, at its own columns.
//  domain    the envelope is kept over [F, c1) only: an empty stack pushes
//            with start F (the first column not yet emitted), a parabola
//            whose start lies past c1-1 is not pushed (:218 with cols -> c1).
//  emission  every later parabola p >= m+1 has D_p(j) >= (m+1-j)^2 for
//            j <= m+1.  The bottom entry (k_b, s_b) owns [s_b, e_b]; its value
//            minus (m+1-j)^2 increases with j, so it is final once
//                keep_old: g_b + (e_b-k_b)^2 <= (m+1-e_b)^2   (strict for take_new)
//            and can no longer change (a later parabola cannot beat it in its
//            range, so it can neither pop it nor start inside it).  Final
//            entries leave the ring (kLrCap per lane, [entry][lane] in shared
//            memory: each lane hits its own bank) and go to a per-row entry
//            list in global scratch; the scan ends when the chunk's last
//            entry is emitted.  A lane whose ring overflows gives its row to
//            the merge-tree kernel (k_rows.cu: row-list mode, or row_done = 2
//            in the default mode, where this kernel takes the rows of sparse
//            planes -- lr_plane -- and k_rows / k_rows_dense the others).
//  fill      lane = column: batches of rows have their lists staged into the
//            idle ring storage (cp.async, all copies in flight), then the warp
//            walks each row with a 32-entry window of the list (entry: column
//            | start << 16, plus the column's nearest row).  Entries starting
//            inside a 128-column block are marked in a 4-word mask (REDUX.OR);
//            lane l owns columns b+4l..b+4l+3, and the owner of column c is
//            the block's first owner plus the marks at or before c (popc).
//            D, sqrt(D), label and nearest column leave with 16-byte stores.
//            A block with 31 or more starts (a dense stretch) is done as one
//            32-column block, lane = column.
//
// tests/lr_model.py is the statement-level model (fuzzed against brute force
// for both tie rules, chunk widths 1..40).
#include <type_traits>

#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kLrCap = 32;               // live entries per lane (ring, power of two)
constexpr int kLrWarps = 4;              // warps per CTA
constexpr uint32_t kLrInfK = 0xFFFFu;    // owner "column" of a featureless row

struct LrSmem {
    uint32_t ks[kLrCap][32];   // column | start << 16
    uint16_t rr[kLrCap][32];   // nearest row of the column (vertical distance in vdist mode)
};

__device__ __forceinline__ const uint16_t* lr_col_ptr(const RowArgs& a, const uint16_t* rowp, int m) {
    if (a.tile_cols >= a.W) return rowp + m;
    const int t = m / a.tile_cols;
    return rowp + t * a.tile_stride + (m - t * a.tile_cols);
}

// Fill one row's columns [c0, c1) from its entry list (column | start << 16,
// plus the column's nearest row), lane = column; shared by k_rows_lr and
// k_rows_pts.  rE / rR are in shared memory.  DONLY: only values are written
// (Drow, optionally Srow; the caller checked LB and NC are null), so a block
// needs no owner per column: D(j) is the minimum of the parabolas of the
// owners around j (each is >= the envelope, and j's owner is among them).
template <int DONLY = 0>  // 0: owners per column; 1: values only, D; 2: values only, D and sqrt D
__device__ __forceinline__ void lr_fill_row(const RowArgs& a, const uint32_t* rE, const uint16_t* rR, int nE,
                                            uint32_t giR, int32_t* Drow, float* Srow, int32_t* Lrow,
                                            int32_t* Nrow, int c0, int c1, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    const int W = a.W;
    const bool vec4 = a.vec;  // 16-byte stores legal (W % 4 == 0, aligned planes)
    auto put = [&](int j, uint32_t d, uint32_t k, uint32_t r) {  // one column, scalar
        const bool inf = k == kLrInfK;
        if (Drow) __stcs(Drow + j, (int32_t)d);
        if (Srow) __stcs(Srow + j, dist_f32(d));
        if (Lrow) __stcs(Lrow + j, inf ? -1 : (int32_t)(r * (uint32_t)W + k));
        if (Nrow) __stcs(Nrow + j, inf ? -1 : (int32_t)k);
    };
    auto put4 = [&](int j, bool fast, uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3) {  // values only
        if (fast || (vec4 && j + 3 < c1)) {
            __stcs(reinterpret_cast<int4*>(Drow + j), make_int4((int)d0, (int)d1, (int)d2, (int)d3));
            if (DONLY == 2)
                __stcs(reinterpret_cast<float4*>(Srow + j),
                       make_float4(dist_f32(d0), dist_f32(d1), dist_f32(d2), dist_f32(d3)));
        } else {
            const uint32_t d[4] = {d0, d1, d2, d3};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (j + t < c1) {
                    __stcs(Drow + j + t, (int32_t)d[t]);
                    if (DONLY == 2) __stcs(Srow + j + t, dist_f32(d[t]));
                }
        }
    };
    auto dval = [&](uint32_t g, uint32_t k, int j) -> uint32_t {
        const int dj = j - (int)k;
        return g == kInfU ? (uint32_t)DFC_INF_I32 : g + (uint32_t)(dj * dj);
    };
    int base = 0;  // entry owning column b
    int b = c0;
    while (b < c1) {
        // window: lane e holds entry base + e; entries 1.. start after b-1
        const int idx = base + lane;
        const uint32_t we = idx < nE ? rE[idx] : FULL;
        const uint32_t wr = idx < nE ? (uint32_t)rR[idx] : kNoRow;
        const int s = (int)(we >> 16);
        const uint32_t wk = we & 0xffffu;
        const uint32_t wav = giR > wr ? giR - wr : wr - giR;
        const uint32_t wg = wk == kLrInfK ? kInfU : wav * wav;
        if (DONLY) {
            // ---- values only, a block of kH x 128 columns whose owners all sit in the
            // window (the usual case on sparse planes): lane l owns columns
            // b + 128 h + 4 l + t (coalesced 16-byte stores per h).  cnt[h] =
            // entries starting at or before b + 128 h, so sub-block h is owned
            // by entries cnt[h] .. cnt[h+1] (warp-uniform), and D(j) is the
            // minimum of THEIR parabolas g + (j - k)^2: each is >= the
            // envelope and j's owner is among them (uint32: an entry that owns
            // a column within 512 of j has a value < 2^31 + 2^26 at j) ----
#ifndef DFC_FILL_KH
#define DFC_FILL_KH 4
#endif
            constexpr int kH = DFC_FILL_KH;  // 128-column sub-blocks per block: 4 or 8
            static_assert(kH == 4 || kH == 8, "one or two REDUX words of four byte counters");
            const int s31 = __shfl_sync(FULL, s, 31);
            if (s31 > b + 128 * kH) {  // the window holds every start up to the block's end
                // cnt[h] = entries (lanes >= 1) starting at or before b + 128 h: an entry
                // counts from sub-block ceil((s - b) / 128) on; one REDUX.ADD of a byte per
                // sub-block (four per word), prefix sums by a multiply (at most 31 entries:
                // no carries)
                const int cf = (s - b + 127) >> 7;  // >= 1 for lanes >= 1 (they start after b)
                int cnt[kH + 1];
                cnt[0] = 0;
                {
                    const uint32_t lo = __reduce_add_sync(FULL, (lane >= 1 && cf <= 4) ? 1u << (8 * (cf - 1)) : 0u);
                    const uint32_t pre = lo * 0x01010101u;
#pragma unroll
                    for (int h = 1; h <= 4; ++h) cnt[h] = (int)((pre >> (8 * (h - 1))) & 0xffu);
                    if (kH == 8) {
                        const uint32_t hi =
                            __reduce_add_sync(FULL, (lane >= 1 && cf > 4 && cf <= 8) ? 1u << (8 * (cf - 5)) : 0u);
                        const uint32_t pre2 = (hi + (pre >> 24)) * 0x01010101u;  // byte k: cnt[4] + n5 + .. + n(5+k)
#pragma unroll
                        for (int h = 5; h <= kH; ++h) cnt[h] = (int)((pre2 >> (8 * (h - 5))) & 0xffu);
                    }
                }
                const bool fast = vec4 && b + 128 * kH <= c1;
                const int j0 = b + 4 * lane;
                auto block = [&](auto FAST) {
                    constexpr bool kFast = decltype(FAST)::value;
                    if (__shfl_sync(FULL, wk, 0) == kLrInfK) {  // featureless row: its only entry
#pragma unroll
                        for (int h = 0; h < kH; ++h) {
                            const uint32_t di = (uint32_t)DFC_INF_I32;
                            put4(j0 + 128 * h, kFast, di, di, di, di);
                        }
                        return;
                    }
                    // the four sub-blocks' first owners up front: eight independent shuffles
                    uint32_t g0[kH];
                    int k0[kH];
#pragma unroll
                    for (int h = 0; h < kH; ++h) {
                        g0[h] = __shfl_sync(FULL, wg, cnt[h]);
                        k0[h] = (int)__shfl_sync(FULL, wk, cnt[h]);
                    }
#pragma unroll
                    for (int h = 0; h < kH; ++h) {
                        const int j = j0 + 128 * h;
                        uint32_t d0, d1, d2, d3;
                        {
                            const uint32_t ge = g0[h];
                            const int dj = j - k0[h];
                            const uint32_t inc = (uint32_t)(2 * dj + 1);
                            d0 = ge + (uint32_t)(dj * dj);
                            d1 = d0 + inc;
                            d2 = d1 + inc + 2u;
                            d3 = d2 + inc + 4u;
                        }
                        for (int e = cnt[h] + 1; e <= cnt[h + 1]; ++e) {  // warp-uniform trip count
                            const uint32_t ge = __shfl_sync(FULL, wg, e);
                            const int dj = j - (int)__shfl_sync(FULL, wk, e);
                            const uint32_t inc = (uint32_t)(2 * dj + 1);
                            const uint32_t v0 = ge + (uint32_t)(dj * dj);
                            const uint32_t v1 = v0 + inc, v2 = v1 + inc + 2u, v3 = v2 + inc + 4u;
                            d0 = min(d0, v0);
                            d1 = min(d1, v1);
                            d2 = min(d2, v2);
                            d3 = min(d3, v3);
                        }
                        put4(j, kFast, d0, d1, d2, d3);
                    }
                };
                if (fast)
                    block(std::true_type{});
                else
                    block(std::false_type{});
                base += cnt[kH];  // the last entry starting at or before the next block's first column
                b += 128 * kH;
                continue;
            }
        }
        const int nin = __popc(__ballot_sync(FULL, lane >= 1 && s <= b + 127));
        if (nin <= 3) {
            // ---- 128-column block with at most 3 owner changes (sparse rows):
            // broadcast the block's owners, each column keeps the last one
            // starting at or before it ----
            const int j = b + 4 * lane;
            uint32_t kc[4], gc[4], rc[4];
            {
                const uint32_t k0 = __shfl_sync(FULL, wk, 0), g0 = __shfl_sync(FULL, wg, 0);
                const uint32_t r0 = __shfl_sync(FULL, wr, 0);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    kc[t] = k0;
                    gc[t] = g0;
                    rc[t] = r0;
                }
            }
            for (int e = 1; e <= nin; ++e) {  // warp-uniform trip count
                const int se = __shfl_sync(FULL, s, e);
                const uint32_t ke = __shfl_sync(FULL, wk, e), ge = __shfl_sync(FULL, wg, e);
                const uint32_t re = __shfl_sync(FULL, wr, e);
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (j + t >= se) {
                        kc[t] = ke;
                        gc[t] = ge;
                        rc[t] = re;
                    }
            }
            const uint32_t d0 = dval(gc[0], kc[0], j), d1 = dval(gc[1], kc[1], j + 1);
            const uint32_t d2 = dval(gc[2], kc[2], j + 2), d3 = dval(gc[3], kc[3], j + 3);
            if (vec4 && j + 3 < c1) {
                if (Drow) __stcs(reinterpret_cast<int4*>(Drow + j), make_int4((int)d0, (int)d1, (int)d2, (int)d3));
                if (Srow)
                    __stcs(reinterpret_cast<float4*>(Srow + j),
                           make_float4(dist_f32(d0), dist_f32(d1), dist_f32(d2), dist_f32(d3)));
                auto lab = [&](uint32_t k, uint32_t r) {
                    return k == kLrInfK ? -1 : (int32_t)(r * (uint32_t)W + k);
                };
                auto nc = [&](uint32_t k) { return k == kLrInfK ? -1 : (int32_t)k; };
                if (Lrow)
                    __stcs(reinterpret_cast<int4*>(Lrow + j), make_int4(lab(kc[0], rc[0]), lab(kc[1], rc[1]),
                                                                       lab(kc[2], rc[2]), lab(kc[3], rc[3])));
                if (Nrow)
                    __stcs(reinterpret_cast<int4*>(Nrow + j), make_int4(nc(kc[0]), nc(kc[1]), nc(kc[2]), nc(kc[3])));
            } else {
                if (j < c1) put(j, d0, kc[0], rc[0]);
                if (j + 1 < c1) put(j + 1, d1, kc[1], rc[1]);
                if (j + 2 < c1) put(j + 2, d2, kc[2], rc[2]);
                if (j + 3 < c1) put(j + 3, d3, kc[3], rc[3]);
            }
            // the next block's first owner: the last entry starting <= b+128
            const int sn = __shfl_sync(FULL, s, nin + 1);
            base += nin + (sn == b + 128 ? 1 : 0);
            b += 128;
        } else if (nin < 31) {
            // ---- 128-column block, 4 columns per lane: the window holds
            // every owner; bit (s-b)&31 of word (s-b)>>5 marks a start ----
            const bool in = lane >= 1 && s <= b + 127;
            const int off = s - b;
            uint32_t Zw[4];
#pragma unroll
            for (int w = 0; w < 4; ++w)
                Zw[w] = __reduce_or_sync(FULL, (in && (off >> 5) == w) ? 1u << (off & 31) : 0u);
            const int w = lane >> 3, bit = (4 * lane) & 31;
            const uint32_t Z = w == 0 ? Zw[0] : w == 1 ? Zw[1] : w == 2 ? Zw[2] : Zw[3];
            const int P = (w >= 1 ? __popc(Zw[0]) : 0) + (w >= 2 ? __popc(Zw[1]) : 0) +
                          (w >= 3 ? __popc(Zw[2]) : 0);
            const int o0 = P + __popc(Z & ((2u << bit) - 1u));
            const int o1 = o0 + (int)((Z >> (bit + 1)) & 1u);
            const int o2 = o1 + (int)((Z >> (bit + 2)) & 1u);
            const int o3 = o2 + (int)((Z >> (bit + 3)) & 1u);
            uint32_t k0 = __shfl_sync(FULL, wk, o0), g0 = __shfl_sync(FULL, wg, o0);
            uint32_t k3 = __shfl_sync(FULL, wk, o3), g3 = __shfl_sync(FULL, wg, o3);
            uint32_t k1 = o1 == o0 ? k0 : k3, g1 = o1 == o0 ? g0 : g3;
            uint32_t k2 = o2 == o3 ? k3 : k0, g2 = o2 == o3 ? g3 : g0;
            if (__any_sync(FULL, o3 - o0 >= 2)) {  // three or more owners in 4 columns
                k1 = __shfl_sync(FULL, wk, o1);
                g1 = __shfl_sync(FULL, wg, o1);
                k2 = __shfl_sync(FULL, wk, o2);
                g2 = __shfl_sync(FULL, wg, o2);
            }
            uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
            if (Lrow) {
                r0 = __shfl_sync(FULL, wr, o0);
                r1 = __shfl_sync(FULL, wr, o1);
                r2 = __shfl_sync(FULL, wr, o2);
                r3 = __shfl_sync(FULL, wr, o3);
            }
            const int j = b + 4 * lane;
            const uint32_t d0 = dval(g0, k0, j), d1 = dval(g1, k1, j + 1);
            const uint32_t d2 = dval(g2, k2, j + 2), d3 = dval(g3, k3, j + 3);
            if (vec4 && j + 3 < c1) {
                if (Drow) __stcs(reinterpret_cast<int4*>(Drow + j), make_int4((int)d0, (int)d1, (int)d2, (int)d3));
                if (Srow)
                    __stcs(reinterpret_cast<float4*>(Srow + j),
                           make_float4(dist_f32(d0), dist_f32(d1), dist_f32(d2), dist_f32(d3)));
                if (Lrow) {
                    auto lab = [&](uint32_t k, uint32_t r) {
                        return k == kLrInfK ? -1 : (int32_t)(r * (uint32_t)W + k);
                    };
                    __stcs(reinterpret_cast<int4*>(Lrow + j), make_int4(lab(k0, r0), lab(k1, r1), lab(k2, r2), lab(k3, r3)));
                }
                if (Nrow) {
                    auto nc = [&](uint32_t k) { return k == kLrInfK ? -1 : (int32_t)k; };
                    __stcs(reinterpret_cast<int4*>(Nrow + j), make_int4(nc(k0), nc(k1), nc(k2), nc(k3)));
                }
            } else {
                if (j < c1) put(j, d0, k0, r0);
                if (j + 1 < c1) put(j + 1, d1, k1, r1);
                if (j + 2 < c1) put(j + 2, d2, k2, r2);
                if (j + 3 < c1) put(j + 3, d3, k3, r3);
            }
            // the next block's first owner: the last entry starting <= b+128
            const int sn = __shfl_sync(FULL, s, min(nin + 1, 31));
            base += nin + ((nin + 1 <= 31 && sn == b + 128) ? 1 : 0);
            b += 128;
        } else {
            // ---- dense stretch: one 32-column block, lane = column ----
            const bool in = lane >= 1 && s <= b + 31;
            const uint32_t Z = __reduce_or_sync(FULL, in ? 1u << (s - b) : 0u);
            const int ow = __popc(Z & ((2u << lane) - 1u));
            const uint32_t k = __shfl_sync(FULL, wk, ow);
            const uint32_t g = __shfl_sync(FULL, wg, ow);
            const uint32_t r = __shfl_sync(FULL, wr, ow);
            const int j = b + lane;
            if (j < c1) put(j, dval(g, k, j), k, r);
            // the next block's first owner: the last entry starting <= b+32
            // (up to 32 entries after base: entry base+32 is read by lane 0)
            const uint32_t s32 = (lane == 0 && base + 32 < nE) ? (rE[base + 32] >> 16) : 0xffffu;
            base += __popc(__ballot_sync(FULL, lane >= 1 && s <= b + 32)) +
                    ((int)__shfl_sync(FULL, s32, 0) <= b + 32 ? 1 : 0);
            b += 32;
        }
    }
}

template <bool TAKE_NEW>
__global__ void __launch_bounds__(32 * kLrWarps, 8) k_rows_lr(RowArgs a, uint32_t* ent, uint16_t* entr, int Ws,
                                                           int C, int* fail_rows, int* fail_count) {
    extern __shared__ uint4 lr_raw[];
    LrSmem& sm = reinterpret_cast<LrSmem*>(lr_raw)[threadIdx.x >> 5];
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int W = a.W;
    const int nchunks = (W + C - 1) / C;
    const int64_t wid = (int64_t)blockIdx.x * kLrWarps + (threadIdx.x >> 5);
    const int64_t band = wid / nchunks;
    if (band * 32 >= a.total_rows) return;  // warp-uniform
    const int c0 = (int)(wid - band * nchunks) * C, c1 = min(c0 + C, W);
    const int64_t row = band * 32 + lane;
    bool active = row < a.total_rows;
    const int img = active ? (int)(row / a.H) : 0;
    if (a.lr_gate) {  // default mode: only the rows of sparse planes
        active = active && lr_plane(a.plane_counts, img, a.H, a.W) && !pts_plane(a.plane_counts, img, a.pts_gate);
        if (!__any_sync(FULL, active)) return;
    }
    const uint32_t i = active ? (uint32_t)(row - (int64_t)img * a.H) : 0u;
    const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;
    const uint16_t* rowp = a.nr + (active ? img * a.nr_img_stride + (int64_t)i * a.Wp : 0);

    // 8 columns of the row (raw: columns past the row end are masked by fix8 at
    // the point of use, so that a prefetch is not consumed as soon as it is
    // issued -- the masking selects would wait on the load)
    auto load8 = [&](int m0) -> uint4 {
        uint4 v = make_uint4(FULL, FULL, FULL, FULL);
        if (active && m0 < W) v = __ldg(reinterpret_cast<const uint4*>(lr_col_ptr(a, rowp, m0)));
        return v;
    };
    auto fix8 = [&](uint4 v, int m0) -> uint4 {
        if (m0 + 8 > W) {  // columns past the row end: no candidate (warp-uniform)
            const int valid = W - m0;  // <= 7 (m0 >= W: already FULL)
            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (2 * t >= valid) w[t] = FULL;
                else if (2 * t + 1 >= valid) w[t] |= 0xffff0000u;
            }
        }
        return v;
    };
    auto half = [](const uint4& v, int t) -> uint32_t {
        const uint32_t w = t < 2 ? (t == 0 ? v.x : v.y) : (t == 2 ? v.z : v.w);
        return w;
    };

    // ---- exact scan bounds: the owners of the columns just left of the chunk
    // and of its last column.  Owners are monotone in j under either tie rule,
    // so every owner of [c0, c1) lies in [owner(c0-1), owner(c1-1)]: only those
    // candidates are scanned.  Each lane searches its own row outward from b in
    // 8-column groups until the nearest unexamined column d has d^2 > best. ----
    auto owner_of = [&](int b) -> int {  // -1: the row has no candidate
        uint32_t best = kInfU;
        int bk = -1;
        auto consider = [&](int k, uint32_t r) {
            if (r == kNoRow) return;
            const uint32_t av = gi > r ? gi - r : r - gi;
            const int h = k - b;
            const uint32_t v = av * av + (uint32_t)(h * h);
            if (v < best || (v == best && (TAKE_NEW ? k > bk : k < bk))) {
                best = v;
                bk = k;
            }
        };
        int lo = b & ~7, hi = lo + 8;  // examined columns [lo, hi)
        bool go = active;
        uint4 v = fix8(load8(lo), lo);
#pragma unroll
        for (int t = 0; t < 8; ++t) consider(lo + t, (half(v, t >> 1) >> (16 * (t & 1))) & 0xffffu);
        for (;;) {
            const int dl = b - lo + 1, dr = hi - b;  // distance of the nearest unexamined column per side
            const bool left = lo > 0 && (uint32_t)(dl * dl) <= best;
            const bool right = hi < W && (uint32_t)(dr * dr) <= best;
            go = go && (left || right);
            if (!__any_sync(FULL, go)) break;
            uint4 vl = make_uint4(FULL, FULL, FULL, FULL), vr = vl;
            if (go && left) vl = load8(lo - 8);
            if (go && right) vr = fix8(load8(hi), hi);
            if (go && left) {
#pragma unroll
                for (int t = 7; t >= 0; --t) consider(lo - 8 + t, (half(vl, t >> 1) >> (16 * (t & 1))) & 0xffffu);
                lo -= 8;
            }
            if (go && right) {
#pragma unroll
                for (int t = 0; t < 8; ++t) consider(hi + t, (half(vr, t >> 1) >> (16 * (t & 1))) & 0xffffu);
                hi += 8;
            }
        }
        return bk;
    };
    int kS = 0, kE = W - 1;
    bool featureless = false;
    if (c0 > 0) {
        kS = owner_of(c0 - 1);
        featureless = kS < 0;
    }
    if (c1 < W) {
        kE = owner_of(c1 - 1);
        featureless = kE < 0;
    }

    // ---- scan ----
    int n = 0, head = 0;                 // ring entries head .. head+n-1
    int tk = 0, ts = 0;                  // top entry
    uint32_t tg = 0;
    int F = c0;                          // first column not yet emitted
    int nout = 0;
    bool done = !active, fail = false;
    const int64_t eoff = active ? row * (int64_t)Ws + c0 : 0;
    uint32_t* eout = ent + eoff;
    uint16_t* rout = entr + eoff;

    // one candidate column: pops, then a push (ring room is checked per group)
    auto cand = [&](int m, uint32_t r) {
        if (r == kNoRow) return;
        const uint32_t av = gi > r ? gi - r : r - gi;
        const uint32_t gm = av * av;
        int start = F;
        while (n > 0) {
            // num = g_m - g_k + m^2 - k^2, |num| < 2^31; ts*den, (c1-1)*den < 2^31
            const int dm = m - tk;
            const int num = (int)gm - (int)tg + dm * (m + tk);
            const int den = 2 * dm;
            const int lim = ts * den;  // start <= js[idx]: pop (:214)
            if (TAKE_NEW ? num <= lim : num < lim) {
                if (--n > 0) {
                    const int idx = (head + n - 1) & (kLrCap - 1);
                    const uint32_t e = sm.ks[idx][lane];
                    tk = (int)(e & 0xffffu);
                    ts = (int)(e >> 16);
                    const uint32_t rk = sm.rr[idx][lane];
                    const uint32_t ak = gi > rk ? gi - rk : rk - gi;
                    tg = ak * ak;
                }
                continue;
            }
            // push iff start <= c1-1 (:218); 0 <= num, quotient < c1 <= 2^15
            if (TAKE_NEW ? num > (c1 - 1) * den : num >= (c1 - 1) * den) return;
            const uint32_t q = small_udiv((uint32_t)num, (uint32_t)den);
            // keep_old: floor(x)+1 ; take_new: ceil(x)   (:205)
            start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * (uint32_t)den)) : (int)q + 1;
            break;
        }
        const int idx = (head + n) & (kLrCap - 1);
        sm.ks[idx][lane] = (uint32_t)m | ((uint32_t)start << 16);
        sm.rr[idx][lane] = (uint16_t)r;
        ++n;
        tk = m;
        ts = start;
        tg = gm;
    };
    // emit final bottom entries (columns <= m scanned); the bottom is read from the ring
    auto emit = [&](int m, bool force) {
        while (n > 0) {
            const uint32_t e = sm.ks[head][lane];
            const int bk = (int)(e & 0xffffu);
            const uint32_t rk = sm.rr[head][lane];
            const int be = n >= 2 ? (int)(sm.ks[(head + 1) & (kLrCap - 1)][lane] >> 16) - 1 : c1 - 1;
            if (!force) {
                const uint32_t ak = gi > rk ? gi - rk : rk - gi;
                const int t = m + 1 - be, dd = be - bk;
                const uint32_t d = ak * ak + (uint32_t)(dd * dd), lim = (uint32_t)(t * t);
                if (TAKE_NEW ? d >= lim : d > lim) break;
            }
            rout[nout] = (uint16_t)rk;
            eout[nout++] = e;
            F = be + 1;
            head = (head + 1) & (kLrCap - 1);
            if (--n == 0) done = true;  // the last entry owns through c1-1
        }
    };

    // ---- scan [kS, kE], each lane at its own columns (8 per 16-byte load) ----
    if (featureless) done = true;
    int m0 = kS & ~7;
    uint4 cur = load8(m0);
    for (;;) {
        const bool mine = !done && m0 <= kE;
        if (!__any_sync(FULL, mine)) break;
        const bool more = mine && m0 + 8 <= kE;
        uint4 nxt = make_uint4(FULL, FULL, FULL, FULL);
        if (more) nxt = load8(m0 + 8);
        cur = fix8(cur, m0);
        if (mine) {
            if ((cur.x & cur.y & cur.z & cur.w) != FULL) {  // any candidate among the 8 columns
                if (n > kLrCap - 8) {  // no room for 8 pushes: the row goes to the merge-tree kernel
                    fail = true;
                    done = true;
                    n = 0;
                    if (a.row_done) a.row_done[row] = 2;  // default mode: k_rows picks it up
                    else fail_rows[atomicAdd(fail_count, 1)] = (int)row;
                } else {
#pragma unroll
                    for (int t = 0; t < 8; ++t) cand(m0 + t, (half(cur, t >> 1) >> (16 * (t & 1))) & 0xffffu);
                }
            }
            if (!done) emit(m0 + 7, false);
        }
        m0 += 8;
        cur = nxt;
    }
    if (active && !fail) {  // no later candidate: everything left is final
        emit(0, true);
        if (F < c1) {  // featureless row
            rout[nout] = kNoRow;
            eout[nout++] = kLrInfK | ((uint32_t)F << 16);
        }
        done = true;
    }
    __syncwarp();

    // ---- fill: lane = column.  Rows are staged in batches: their entry lists
    // (cp.async, 16-byte granules, L2) into the now idle ring storage ----
    constexpr int kStage = kLrCap * 32;                // staging capacity (entries)
    const int myall = (active && !fail) ? nout : 0;
    const int myn = myall <= kStage ? myall : 0;      // longer lists: direct pass below
    const int maxn = (int)__reduce_max_sync(FULL, (unsigned)myn);
    const int S = max(32, (maxn + 31) & ~31);          // staging stride per row (<= kStage)
    const int rpb = min(32, kStage / S);               // rows per batch
    uint32_t* sE = &sm.ks[0][0];
    uint16_t* sR = &sm.rr[0][0];
    const uint32_t sE_addr = (uint32_t)__cvta_generic_to_shared(sE);
    const uint32_t sR_addr = (uint32_t)__cvta_generic_to_shared(sR);
    for (int r0 = 0; r0 < 32; r0 += rpb) {
        const int r1 = min(32, r0 + rpb);
        __syncwarp();
        for (int rho = r0; rho < r1; ++rho) {
            const int nE = __shfl_sync(FULL, myn, rho);
            const int64_t off = (band * 32 + rho) * (int64_t)Ws + c0;
            const int slot = (rho - r0) * S;
            for (int q = lane; 4 * q < nE; q += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sE_addr + 4u * (slot + 4 * q)),
                             "l"(ent + off + 4 * q));
            for (int q = lane; 8 * q < nE; q += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sR_addr + 2u * (slot + 8 * q)),
                             "l"(entr + off + 8 * q));
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncwarp();
        for (int rho = r0; rho < r1; ++rho) {
            const int nE = __shfl_sync(FULL, myn, rho);
            if (nE == 0) continue;  // failed (k_rows recomputes it) or no row
            const uint32_t giR = __shfl_sync(FULL, gi, rho);
            const int64_t rowR = band * 32 + rho;
            const int imgR = (int)(rowR / a.H);
            const int64_t iR = rowR - (int64_t)imgR * a.H;
            int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + imgR * a.sD) + iR * W : nullptr;
            float* Srow = a.S ? reinterpret_cast<float*>(a.S + imgR * a.sS) + iR * W : nullptr;
            int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + imgR * a.sL) + iR * W : nullptr;
            int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + imgR * a.sN) + iR * W : nullptr;
            const uint32_t* rE = sE + (rho - r0) * S;
            const uint16_t* rR = sR + (rho - r0) * S;
            if (Drow && !Srow && !Lrow && !Nrow)
                lr_fill_row<1>(a, rE, rR, nE, giR, Drow, Srow, Lrow, Nrow, c0, c1, lane);
            else
                lr_fill_row<0>(a, rE, rR, nE, giR, Drow, Srow, Lrow, Nrow, c0, c1, lane);
        }
    }
    // rows whose list exceeds the staging capacity (chunks wider than kStage
    // columns with dense envelopes): 32-column blocks straight from L2
    const uint32_t big = __ballot_sync(FULL, myall > kStage);
    for (uint32_t bm = big; bm; bm &= bm - 1) {
        const int rho = __ffs(bm) - 1;
        const int nE = __shfl_sync(FULL, myall, rho);
        const uint32_t giR = __shfl_sync(FULL, gi, rho);
        const int64_t rowR = band * 32 + rho;
        const int imgR = (int)(rowR / a.H);
        const int64_t iR = rowR - (int64_t)imgR * a.H;
        int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + imgR * a.sD) + iR * W : nullptr;
        float* Srow = a.S ? reinterpret_cast<float*>(a.S + imgR * a.sS) + iR * W : nullptr;
        int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + imgR * a.sL) + iR * W : nullptr;
        int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + imgR * a.sN) + iR * W : nullptr;
        const int64_t off = rowR * (int64_t)Ws + c0;
        int base = 0;
        for (int b = c0; b < c1; b += 32) {
            const int idx = base + lane;
            const uint32_t we = idx < nE ? __ldcg(ent + off + idx) : FULL;
            const uint32_t wr = idx < nE ? (uint32_t)__ldcg(entr + off + idx) : kNoRow;
            const int s = (int)(we >> 16);
            const bool in = lane >= 1 && s <= b + 31;
            const uint32_t Z = __reduce_or_sync(FULL, in ? 1u << (s - b) : 0u);
            const int ow = __popc(Z & ((2u << lane) - 1u));
            const uint32_t ke = __shfl_sync(FULL, we, ow);
            const uint32_t kr = __shfl_sync(FULL, wr, ow);
            const int j = b + lane;
            if (j < c1) {
                const uint32_t k = ke & 0xffffu;
                const bool inf = k == kLrInfK;
                const uint32_t av = giR > kr ? giR - kr : kr - giR;
                const int dj = j - (int)k;
                const uint32_t d = inf ? (uint32_t)DFC_INF_I32 : av * av + (uint32_t)(dj * dj);
                if (Drow) __stcs(Drow + j, (int32_t)d);
                if (Srow) __stcs(Srow + j, dist_f32(d));
                if (Lrow) __stcs(Lrow + j, inf ? -1 : (int32_t)(kr * (uint32_t)W + k));
                if (Nrow) __stcs(Nrow + j, inf ? -1 : (int32_t)k);
            }
            const uint32_t s32 = (lane == 0 && base + 32 < nE) ? (__ldcg(ent + off + base + 32) >> 16) : 0xffffu;
            base += __popc(__ballot_sync(FULL, lane >= 1 && s <= b + 32)) +
                    ((int)__shfl_sync(FULL, s32, 0) <= b + 32 ? 1 : 0);
        }
    }
}

// Rows the segment kernel still has to do in the default mode: not written by
// k_rows_dense (flag 1), and not a sparse-plane row k_rows_lr completed
// (sparse plane, flag != 2).  Appended to a list (any order).
__global__ void k_rows_rest(const uint8_t* row_done, const unsigned long long* counts, int64_t total_rows,
                            int H, int W, bool lr_gate, bool pts_gate, int* list, int* count) {
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < total_rows;
         row += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t rd = row_done[row];
        const int img = (int)(row / H);
        const bool mine = !pts_plane(counts, img, pts_gate) &&
                          (rd == 2 || (rd == 0 && !(lr_gate && lr_plane(counts, img, H, W))));
        const unsigned m = __ballot_sync(__activemask(), mine);
        if (m == 0) continue;
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(count, __popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (mine) list[base + __popc(m & ((1u << lane) - 1u))] = (int)row;
    }
}

// Rows k_rows_lr flagged as overflowed (row_done == 2), appended to a list
// once each (mode 5's fallback list: at most total_rows entries).
__global__ void k_rows_failed(const uint8_t* row_done, int64_t total_rows, int* list, int* count) {
    for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < total_rows;
         row += (int64_t)gridDim.x * blockDim.x) {
        const bool mine = row_done[row] == 2;
        const unsigned m = __ballot_sync(__activemask(), mine);
        if (m == 0) continue;
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(count, __popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (mine) list[base + __popc(m & ((1u << lane) - 1u))] = (int)row;
    }
}

// Object pixels of a (possibly column-tiled) nearest-row plane: cells whose
// nearest object row is their own row (the sparse-plane gate of
// dfc_rows_from_nr_u16, where no column pass of the whole image ran here).
__global__ void k_nr_count(RowArgs a, unsigned long long* count) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x; i < a.total_rows; i += gridDim.x) {
        const uint16_t* rowp = a.nr + i * a.Wp;
        for (int j = threadIdx.x; j < a.W; j += blockDim.x) c += __ldg(lr_col_ptr(a, rowp, j)) == (uint32_t)(i + a.row0);
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

template <bool TAKE_NEW>
inline const void* lr_kernel_ptr() {
    return (const void*)k_rows_lr<TAKE_NEW>;
}

inline int lr_smem_bytes() { return kLrWarps * (int)sizeof(LrSmem); }

}  // namespace dfc
