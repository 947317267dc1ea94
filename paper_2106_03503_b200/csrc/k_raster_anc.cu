// k_raster_anc.cu -- the row pass of config 4's approximate transforms by
// ANCHORED SEGMENTS (the k_rows_anc.cu scheme), replacing k_raster's outward
// window search for chessboard and chamfer-3-4.
//
// Same maps as the reference's two-pass raster scans cityblock_sequential
// (propagation.cpp:16-34, 90-95) and chamfer34 (propagation.cpp:60-88,
// 104-109), and the chessboard oracle (proj/tests/oracles.hpp:52-55), through
// the separable closed forms of k_raster.cu (a_k = vertical pixel distance to
// the nearest object in column k):
//     city-block  = min_k  a_k + |j-k|
//     chessboard  = min_k  max(a_k, |j-k|)
//     chamfer-3-4 = min_k  3 max(a_k,|j-k|) + min(a_k,|j-k|) = min_k max(3 a_k + h, a_k + 3 h)
//
//  city-block  lane = column of a 32-column segment: min_k (a_k - k) + j over
//              k <= j and min_k (a_k + k) - j over k >= j, as warp prefix /
//              suffix minima plus per-segment carries (one warp scans the
//              segment minima of the row).
//  chessboard, chamfer
//              the smallest minimiser of either family is monotone in j (the
//              single-crossing property of these piecewise-linear shapes;
//              tests/test_oracle.py::test_raster_argmin_monotone{,_synthetic}), so
//              every minimiser a segment needs lies in [owner(j0), owner(j0+32)].
//              Owners every 32 columns come from a divide and conquer over the
//              segment index (lane = candidate, REDUX min), both families in the
//              same level loop; then lane = column scans its segment's range.
//              An object pixel on the row (a = 0) owns itself (value 0), and a
//              segment of object pixels is written directly.
// One CTA (8 warps) per row, grid-stride; coalesced 4-byte stores.
#include <type_traits>

#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kRaWarps = 8;
constexpr int kRaMaxW = 16384;
constexpr int kRaBig = 0x1fffffff;   // a_k of a column without objects (3 kRaBig + h fits int32)
constexpr int kRaNone = 0x7fffffff;

__host__ __device__ __forceinline__ int ra_segs(int W) { return (W + 31) >> 5; }
__host__ __device__ __forceinline__ int ra_gwords(int W) { return (W + 3) & ~3; }
// 16-bit variant (rows and columns <= 8192): a_k as uint16 (kRa16Big for none),
// so that two candidates share one SIMD instruction (VIMNMX.U16x2 / VIADD.16x2);
// every value fits: chessboard <= 8191 < kRa16Big, chamfer <= 32764 <
// 3 kRa16Big <= chamfer of a column without objects <= 57340 < 2^16.
constexpr int kRa16Big = 16383;
constexpr int kRa16MaxDim = 8192;
// words: a (gw, or gw/2 + 4 for uint16), owners of both families (2 (S+1)),
// object bits, segment minima / carries (4 S), parts (4 NW)
inline int ra_smem_bytes(int W, bool p16) {
    const int S = ra_segs(W);
    return ((p16 ? ra_gwords(W) / 2 + 4 : ra_gwords(W)) + 2 * (S + 1) + 5 * S + 4 * kRaWarps) * 4;
}

struct RaInf {
    __device__ __forceinline__ static int f(int a, int h) { return max(a, h); }
};
struct RaCham {
    __device__ __forceinline__ static int f(int a, int h) { return max(3 * a + h, a + 3 * h); }
};

// Minimum of F over the candidates [lo, hi] (possibly empty: kRaNone) for
// column j, and its smallest minimiser: lane = candidate, then REDUX minima.
template <class F, class T>
__device__ __forceinline__ int ra_owner(const T* av, int j, int lo, int hi, int lane, int& col) {
    int best = kRaNone, bk = lo;
    for (int k = lo + lane; k <= hi; k += 32) {
        const int v = F::f((int)av[k], abs(j - k));
        if (v < best) {
            best = v;
            bk = k;
        }
    }
    const int m = __reduce_min_sync(0xffffffffu, best);
    col = (int)__reduce_min_sync(0xffffffffu, best == m ? (unsigned)bk : 0xFFFFFFFFu);
    return m;
}

// Both families' owners for column j over the union of their ranges [lo, hi]
// (uint16 a_k: rows and columns <= 8192), scanned as the even-aligned superset
// [lo & ~1, hi | 1]: an extra candidate can neither go below the minimum nor
// tie it (it would then be a smaller global minimiser than the owner, which
// lies in the range).  Lane = a pair of candidates (one 4-byte load); a
// candidate's key is value << 13 | k, so that one min keeps the smallest
// minimiser and one REDUX yields value and column.  Empty range: kRaNone.
__device__ __forceinline__ void ra_owner2_16(const uint16_t* av, int j, int lo, int hi, int lane, int& mi,
                                             int& ci, int& mc, int& cc) {
    uint32_t bi = 0xffffffffu, bc = 0xffffffffu;
    for (int k = (lo & ~1) + 2 * lane; k <= hi; k += 64) {
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(av + k);
        const int a0 = (int)(a2 & 0xffffu), a1 = (int)(a2 >> 16);
        const int h0 = abs(j - k), h1 = abs(j - k - 1);
        bi = min(bi, ((uint32_t)max(a0, h0) << 13) | (uint32_t)k);
        bi = min(bi, ((uint32_t)max(a1, h1) << 13) | (uint32_t)(k + 1));
        bc = min(bc, ((uint32_t)max(3 * a0 + h0, a0 + 3 * h0) << 13) | (uint32_t)k);
        bc = min(bc, ((uint32_t)max(3 * a1 + h1, a1 + 3 * h1) << 13) | (uint32_t)(k + 1));
    }
    bi = __reduce_min_sync(0xffffffffu, bi);
    bc = __reduce_min_sync(0xffffffffu, bc);
    mi = bi == 0xffffffffu ? kRaNone : (int)(bi >> 13);
    ci = (int)(bi & 8191u);
    mc = bc == 0xffffffffu ? kRaNone : (int)(bc >> 13);
    cc = (int)(bc & 8191u);
}

// Chessboard and chamfer minima for column j over the union of their ranges
// [lo, hi], scanned as its aligned superset [lo & ~3, hi | 3] (extra
// candidates cannot go below a minimum the range attains; the padding past W
// holds kRaBig): one load and one |j - k| for both families, 16-byte loads.
__device__ __forceinline__ void ra_scan2(const int* av, int j, int lo, int hi, int& linf, int& lch) {
    int bi = kRaNone, bc = kRaNone;
    for (int k = lo & ~3; k <= hi; k += 4) {
        const int4 q = *reinterpret_cast<const int4*>(av + k);
        const int aa[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int h = abs(j - k - t), m = max(aa[t], h);
            bi = min(bi, m);
            bc = min(bc, 2 * m + (aa[t] + h));  // 3 max + min
        }
    }
    linf = bi;
    lch = bc;
}

// The same over uint16 a_k, two candidates per SIMD instruction: the superset
// [lo & ~7, hi | 7], 16-byte loads of 8 candidates.
__device__ __forceinline__ void ra_scan2_16(const uint16_t* av, int j, int lo, int hi, int& linf, int& lch) {
    uint32_t bi = 0xffffffffu, bc = 0xffffffffu;
    for (int k = lo & ~7; k <= hi; k += 8) {
        const uint4 q = *reinterpret_cast<const uint4*>(av + k);
        const uint32_t aa[4] = {q.x, q.y, q.z, q.w};
        // (j - k, j - k - 1) as signed 16-bit halves, then 2 less per pair
        uint32_t d2 = (uint32_t)((j - k) & 0xffff) | ((uint32_t)((j - k - 1) & 0xffff) << 16);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t h2 = __vmaxs2(d2, __vsub2(0u, d2));  // |j - k|
            const uint32_t m = __vmaxu2(aa[t], h2);
            bi = __vminu2(bi, m);
            bc = __vminu2(bc, __vadd2(__vadd2(m, m), __vadd2(aa[t], h2)));  // 3 max + min
            d2 = __vsub2(d2, 0x00020002u);
        }
    }
    linf = (int)min(bi & 0xffffu, bi >> 16);
    lch = (int)min(bc & 0xffffu, bc >> 16);
}

template <bool P16>
__global__ void __launch_bounds__(32 * kRaWarps, 6) k_raster_anc(RasterArgs a) {
    using T = typename std::conditional<P16, uint16_t, int>::type;
    extern __shared__ uint4 rasm[];
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int NW = kRaWarps;
    const int W = a.W;
    const int S = ra_segs(W);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    T* av = reinterpret_cast<T*>(rasm);
    int* ancI = reinterpret_cast<int*>(rasm) + (P16 ? ra_gwords(W) / 2 + 4 : ra_gwords(W));  // [S + 1] chessboard owners
    int* ancC = ancI + S + 1;       // [S + 1] chamfer owners
    uint32_t* zb = reinterpret_cast<uint32_t*>(ancC + S + 1);  // [S] object pixels on the row
    int* m1 = reinterpret_cast<int*>(zb + S);  // [S] min (a_k - k) per segment -> exclusive prefix min
    int* m2 = m1 + S;                          // [S] min (a_k + k) per segment -> exclusive suffix min
    int* c1 = m2 + S;                          // [S]
    int* c2 = c1 + S;                          // [S]
    int* pv = c2 + S;                          // [2 NW] partial minima (both families)
    int* pk = pv + 2 * NW;                     // [2 NW] their columns
    int P = 1;
    while (P < S) P <<= 1;

    for (int64_t i64 = blockIdx.x; i64 < a.H; i64 += gridDim.x) {
        const int i = (int)i64;
        const uint16_t* rowp = a.nr + (int64_t)i * a.Wp;
        const int bb = i >> 5, br = i & 31;
        const uint32_t upmask = 0xffffffffu >> (31 - br);

        // ---- stage a_k, the object bits and the segment minima of a_k -/+ k ----
        bool any = false;
        for (int q0 = warp * 32; 4 * q0 < W; q0 += 32 * NW) {  // warp-uniform trip count
            const int q = q0 + lane;
            int d[4] = {kRaBig, kRaBig, kRaBig, kRaBig};
            if (4 * q < W && a.bmask) {  // band source: the band's mask (object = nonzero) and carries
                const int64_t off = (int64_t)bb * a.Wp;
                const uint4 m4 = __ldg(reinterpret_cast<const uint4*>(a.bmask + off) + q);
                const uint2 a2 = __ldg(reinterpret_cast<const uint2*>(a.babove + off) + q);
                const uint2 b2 = __ldg(reinterpret_cast<const uint2*>(a.bbelow + off) + q);
                const uint32_t mm[4] = {m4.x, m4.y, m4.z, m4.w};
                const uint32_t ca[4] = {a2.x & 0xffffu, a2.x >> 16, a2.y & 0xffffu, a2.y >> 16};
                const uint32_t cb[4] = {b2.x & 0xffffu, b2.x >> 16, b2.y & 0xffffu, b2.y >> 16};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t up = mm[t] & upmask, dn = mm[t] >> br;
                    const int du = up ? br - 31 + (int)__clz(up) : (ca[t] == kNoRow ? kRaBig : i - (int)ca[t]);
                    const int dd = dn ? __ffs(dn) - 1 : (cb[t] == kNoRow ? kRaBig : (int)cb[t] - i);
                    if (4 * q + t < W) d[t] = min(du, dd);
                }
            } else if (4 * q < W) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(rowp) + q);
                const uint32_t r[4] = {v.x & 0xffffu, v.x >> 16, v.y & 0xffffu, v.y >> 16};
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (4 * q + t < W && r[t] != kNoRow) d[t] = (uint32_t)i > r[t] ? i - (int)r[t] : (int)r[t] - i;
            }
            uint32_t z = 0;
            int x1 = kRaNone, x2 = kRaNone;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = 4 * q + t;
                any |= d[t] < kRaBig;
                z |= (uint32_t)(d[t] == 0 || j >= W) << t;
                if (j < W) {
                    x1 = min(x1, d[t] - j);
                    x2 = min(x2, d[t] + j);
                }
            }
            if (4 * q < W) {
                if (P16) {
#pragma unroll
                    for (int t = 0; t < 4; ++t) d[t] = min(d[t], kRa16Big);
                    reinterpret_cast<uint2*>(av)[q] = make_uint2((uint32_t)d[0] | ((uint32_t)d[1] << 16),
                                                                 (uint32_t)d[2] | ((uint32_t)d[3] << 16));
                } else {
                    reinterpret_cast<int4*>(av)[q] = make_int4(d[0], d[1], d[2], d[3]);
                }
            }
            z <<= 4 * (lane & 7);
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                z |= __shfl_xor_sync(FULL, z, o);
                x1 = min(x1, __shfl_xor_sync(FULL, x1, o));
                x2 = min(x2, __shfl_xor_sync(FULL, x2, o));
            }
            if ((lane & 7) == 0 && (q >> 3) < S) {
                zb[q >> 3] = z;
                m1[q >> 3] = x1;
                m2[q >> 3] = x2;
            }
        }
        if (P16 && tid < 8) av[ra_gwords(W) + tid] = (T)kRa16Big;  // the superset scan reads up to 8 past
        any = __syncthreads_or(any);
        int32_t* crow = a.city ? a.city + (int64_t)i * W : nullptr;
        int32_t* brow = a.chess ? a.chess + (int64_t)i * W : nullptr;
        int32_t* mrow = a.cham ? a.cham + (int64_t)i * W : nullptr;
        if (!any) {  // featureless image: all infinite (test_propagation.cpp:73-78)
            for (int j = tid; j < W; j += 32 * NW) {
                if (crow) __stcs(crow + j, DFC_INF_I32);
                if (brow) __stcs(brow + j, DFC_INF_I32);
                if (mrow) __stcs(mrow + j, DFC_INF_I32);
            }
            __syncthreads();
            continue;
        }

        // ---- city-block carries: exclusive prefix min of m1, suffix min of m2 (warp 0) ----
        if (warp == 0) {
            const int per = (S + 31) / 32, b0 = lane * per, b1 = min(b0 + per, S);
            int f = kRaNone, g = kRaNone;
            for (int b = b0; b < b1; ++b) f = min(f, m1[b]);
            for (int b = b0; b < b1; ++b) g = min(g, m2[b]);
            int fin = f, gin = g;  // inclusive scans over the lanes' chunk minima
            for (int o = 1; o < 32; o <<= 1) {
                const int uf = __shfl_up_sync(FULL, fin, o), dg = __shfl_down_sync(FULL, gin, o);
                if (lane >= o) fin = min(fin, uf);
                if (lane + o < 32) gin = min(gin, dg);
            }
            int cf = __shfl_up_sync(FULL, fin, 1), cg = __shfl_down_sync(FULL, gin, 1);
            if (lane == 0) cf = kRaNone;
            if (lane == 31) cg = kRaNone;
            for (int b = b0; b < b1; ++b) {
                c1[b] = cf;
                cf = min(cf, m1[b]);
            }
            for (int b = b1 - 1; b >= b0; --b) {
                c2[b] = cg;
                cg = min(cg, m2[b]);
            }
        }

        // ---- owners at every 32nd column, both families: levels of a divide and
        // conquer over [0, P] (index >= S stands for owner(W) := W - 1; index 0
        // last, lower bound 0); an object pixel on the row owns itself ----
        if (tid == 0) {
            ancI[S] = W - 1;
            ancC[S] = W - 1;
        }
        auto on_row = [&](int j) { return (zb[j >> 5] >> (j & 31)) & 1u; };
        for (int step = P >> 1; step >= 0; step >>= 1) {
            const bool last = step == 0;
            const int s0 = last ? 0 : step, ds = last ? 1 : 2 * step;
            const int n = last ? 1 : (S - step + ds - 1) >> (__ffs(ds) - 1);
            if (n <= 0) continue;
            __syncthreads();
            auto bounds = [&](const int* anc, int s, int& lo, int& hi) {
                lo = (last || s - step == 0) ? 0 : anc[s - step];
                hi = last ? (S > 1 ? anc[1] : W - 1) : (s + step >= S ? W - 1 : anc[s + step]);
            };
            if (n >= NW) {
                for (int t = warp; t < n; t += NW) {
                    const int s = s0 + t * ds, j = 32 * s;
                    int ci = j, cc = j;
                    if (!on_row(j)) {
                        int lo, hi;
                        if constexpr (P16) {
                            int lo2, hi2, mi, mc;
                            bounds(ancI, s, lo, hi);
                            bounds(ancC, s, lo2, hi2);
                            ra_owner2_16(av, j, min(lo, lo2), max(hi, hi2), lane, mi, ci, mc, cc);
                        } else {
                            bounds(ancI, s, lo, hi);
                            ra_owner<RaInf>(av, j, lo, hi, lane, ci);
                            bounds(ancC, s, lo, hi);
                            ra_owner<RaCham>(av, j, lo, hi, lane, cc);
                        }
                    }
                    if (lane == 0) {
                        ancI[s] = ci;
                        ancC[s] = cc;
                    }
                }
            } else {
                const int q = NW / n;
                const int t = warp / q, part = warp - t * q;
                int mi = kRaNone, mc = kRaNone, ci = 0, cc = 0;
                if (t < n) {
                    const int s = s0 + t * ds, j = 32 * s;
                    if (on_row(j)) {
                        if (part == 0) {
                            mi = mc = 0;
                            ci = cc = j;
                        }
                    } else if constexpr (P16) {
                        int lo, hi, lo2, hi2;
                        bounds(ancI, s, lo, hi);
                        bounds(ancC, s, lo2, hi2);
                        lo = min(lo, lo2);
                        hi = max(hi, hi2);
                        const int c = (hi - lo + q) / q, plo = lo + part * c;
                        ra_owner2_16(av, j, plo, min(hi, plo + c - 1), lane, mi, ci, mc, cc);
                    } else {
                        int lo, hi;
                        bounds(ancI, s, lo, hi);
                        int c = (hi - lo + q) / q, plo = lo + part * c;
                        mi = ra_owner<RaInf>(av, j, plo, min(hi, plo + c - 1), lane, ci);
                        bounds(ancC, s, lo, hi);
                        c = (hi - lo + q) / q;
                        plo = lo + part * c;
                        mc = ra_owner<RaCham>(av, j, plo, min(hi, plo + c - 1), lane, cc);
                    }
                }
                if (lane == 0) {
                    pv[warp] = mi;
                    pk[warp] = ci;
                    pv[NW + warp] = mc;
                    pk[NW + warp] = cc;
                }
                __syncthreads();
                if (tid < 2 * n) {  // thread f * n + t: family f of anchor t
                    const int f = tid / n, tt = tid - f * n;
                    int bm = kRaNone, bc = 0;
                    for (int p = 0; p < q; ++p) {  // ascending column ranges: first minimum
                        const int v = pv[f * NW + tt * q + p];
                        if (v < bm) {
                            bm = v;
                            bc = pk[f * NW + tt * q + p];
                        }
                    }
                    (f == 0 ? ancI : ancC)[s0 + tt * ds] = bc;
                }
            }
            if (last) break;
        }
        __syncthreads();

        // ---- segments: lane = column ----
        for (int s = warp; s < S; s += NW) {
            const int j = 32 * s + lane;
            const bool in = j < W;
            int l1, linf, lch;
            if (zb[s] == 0xffffffffu) {  // every column an object pixel on the row
                l1 = linf = lch = 0;
            } else {
                const int aj = in ? (int)av[j] : kRaBig;
                int p = in ? aj - j : kRaNone, u = in ? aj + j : kRaNone;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int up = __shfl_up_sync(FULL, p, o), dn = __shfl_down_sync(FULL, u, o);
                    if (lane >= o) p = min(p, up);
                    if (lane + o < 32) u = min(u, dn);
                }
                l1 = min(min(p, c1[s]) + j, min(u, c2[s]) - j);
                const int lo = min(ancI[s], ancC[s]), hi = max(ancI[s + 1], ancC[s + 1]);
                if constexpr (P16)
                    ra_scan2_16(av, j, lo, hi, linf, lch);
                else
                    ra_scan2(av, j, lo, hi, linf, lch);
            }
            if (in) {
                if (crow) __stcs(crow + j, l1);
                if (brow) __stcs(brow + j, linf);
                if (mrow) __stcs(mrow + j, lch);
            }
        }
        __syncthreads();
    }
}

}  // namespace dfc
