// k_rows_band.cu -- stage 2 for SPARSE planes (object pixels < 1/256, C5):
// per band of 32 rows, only the columns that can own a pixel of the band
// enter the row envelopes.
//
// Same result as k_rows.cu / k_rows_lr.cu (envelope_rows / meijster_scan /
// voronoi label assembly, exact_edt.cpp:190-283, :362-369).  The reference's
// stack algorithm (exact_edt.cpp:208-223) visits every column of every row;
// on a sparse plane nearly all of those parabolas are dominated.  Which
// columns can matter is decided once per band of 32 rows:
//
//  candidates  the owner of pixel (i, j) of band b [i0, i1] is a nearest object
//              pixel s* = (r*, k*).  If r* < i0, s* is also nearest among the
//              objects above the band; its Voronoi cell among those (convex,
//              s* inside) then crosses the line i = i0, and s* is the carry
//              above of column k* (a lower object in the same column would be
//              nearer).  So the parabola (i0 - above_k*)^2 + (x - k*)^2 touches
//              the lower envelope over REAL x of the band's carry-above
//              parabolas: the point (k*, H_k*), H_k = (i0 - above_k)^2 + k^2,
//              lies on the lower convex hull of those points (collinear points
//              kept, for ties).  Likewise below the band at i1, and otherwise
//              column k* holds an object pixel inside the band.  Any superset
//              is exact (the row pass evaluates each candidate's true g_k(i)),
//              so the hulls are taken per window of 1024 columns (a hull point
//              of the row is a hull point of every window holding it):
//  k_band_hull warp = (plane, band, side, window); lane = 32 columns: monotone
//              chain with the stack as a 32-bit mask, then 5 levels of bridge
//              merges (walk the lower common tangent) inside the warp; the
//              side-above warps also add the band's object columns.  Output:
//              candidate bit masks [plane][band][side][W/32].  C5: ~640
//              candidates per band out of 32768 columns.
//  k_band_rows warp = (plane, band), lane = row: the reference's stack algorithm
//              over the band's candidates only (g from the band mask and the
//              carries, the upper row on ties, exact_edt.cpp:351), the top
//              kBandCap entries in a shared-memory ring that spills its bottom
//              to the row's list in global memory and reloads from it -- the
//              stack is unbounded, no row needs a fallback.  The final stack is
//              the row's owner list (column | start << 16, nearest row).
//  k_rows_fill warp = row: the list staged in shared memory (cp.async), then
//              the shared lr_fill_row (k_rows_lr.cu): lane = column, 16-byte
//              streaming stores -- the HBM-bound part (C5: 4 B/px).
//
// tests/band_model.py is the statement-level model (fuzzed against brute
// force for both tie rules with small windows, lanes and ring capacities).
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kHullWarps = 2;
constexpr int kHullCap = 64;        // stack entries per hull window
constexpr int kBandWarps = 2;       // k_band_rows: bands per CTA
constexpr int kBandCap = 32;        // ring entries per lane (power of two)
constexpr int kFillWarps = 4;
constexpr int kFillCap = 1536;      // list entries staged per warp (k_rows_fill)

struct BandArgs {
    const uint32_t* bmask;   // [img][nb][Wp] bit r = row 32 b + r nonzero
    const uint16_t* above;   // [plane][nb][Wp] nearest object row above the band (kNoRow: none)
    const uint16_t* below;   // [plane][nb][Wp] nearest object row below the band
    uint32_t* cand;          // [plane][nb][2][Ww] candidate columns (side 0 above + band, 1 below)
    const unsigned long long* counts;  // object pixels per plane
    uint32_t* ent;           // per row list: column | start << 16, at row * Ws
    uint16_t* entr;          // the entries' nearest object rows
    int* nent;               // entries per row
    int64_t Ws;              // list stride per row (entries)
    int H, W, Wp, nb, Ww, n_img, pol0, nplanes;
    // row stripes (the sharded path): local band b is global band band0 + b of
    // an image of Hg rows; plane p's local rows are [0, H).  Single images:
    // band0 = 0, Hg = H.
    int band0, Hg;
    int win;                 // k_band_hull window: ceil(W / 32) rounded up to 32 (<= 1024)
    bool pts_gate;           // point planes belong to k_rows_pts
    bool all_planes;         // every plane (the sharded path), not only the sparse ones
};

// The planes this path owns: sparse, not a point plane.
__device__ __forceinline__ bool band_plane(const BandArgs& a, int p) {
    return a.all_planes || (lr_plane(a.counts, p, a.Hg, a.W) && !pts_plane(a.counts, p, a.pts_gate));
}

// ---------------------------------------------------------------- hull filter
// warp = (plane, band, side); lane = a window of `win` columns (the 32 windows
// cover the row).  Each lane runs the monotone chain over its window (stack in
// shared memory, top two entries cached in registers); then 5 levels of bridge
// merges join the windows' hulls into the row's hull: a merge walks the lower
// common tangent from the left group's last and the right group's first
// vertex, trimming each window's surviving range [lo, hi) of its stack.  A
// window whose stack would exceed kHullCap entries contributes every valid
// column instead and sits out the merges (still a superset).
struct HullSmem {
    int32_t h[kHullCap][32];    // H of the stack entries (< 2^31, see below)
    uint16_t c[kHullCap][32];   // their column offsets in the window
    int lo[32], hi[32];         // surviving range of each window's stack
};

__global__ void __launch_bounds__(32 * kHullWarps) k_band_hull(BandArgs a) {
    __shared__ HullSmem smem[kHullWarps];
    HullSmem& sm = smem[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int64_t task = (int64_t)blockIdx.x * kHullWarps + (threadIdx.x >> 5);
    if (task >= (int64_t)a.nplanes * a.nb * 2) return;
    const int side = (int)(task & 1);
    const int64_t pb = task >> 1;
    const int p = (int)(pb / a.nb), b = (int)(pb - (int64_t)p * a.nb);
    if (!band_plane(a, p)) return;  // warp-uniform
    const int gb = a.band0 + b;      // global band
    const int line = side ? min(32 * gb + 31, a.Hg - 1) : 32 * gb;
    const int WIN = a.win;
    const int k0 = lane * WIN, k1 = min(a.W, k0 + WIN);
    const uint16_t* car = (side ? a.below : a.above) + ((int64_t)p * a.nb + b) * a.Wp;
    // H_k = d^2 + k^2 <= (rows-1)^2 + (cols-1)^2 <= DFC_MAX_SQDIST < 2^31: int32;
    // differences fit int32, times column differences (< 2^15): one IMAD.WIDE
    auto above_seg = [](int ka, int Ha, int kb, int Hb, int kc, int Hc) {
        return (long long)(Hb - Ha) * (kc - kb) > (long long)(Hc - Hb) * (kb - ka);
    };
    // 32 carries of columns [c0, c0 + 32) (kNoRow past the row end)
    auto load32 = [&](int c0, uint32_t (&w)[16]) {
        if (c0 + 32 <= a.Wp) {
            const uint4* q = reinterpret_cast<const uint4*>(car + c0);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint4 x = __ldg(q + v);
                w[4 * v] = x.x; w[4 * v + 1] = x.y; w[4 * v + 2] = x.z; w[4 * v + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const uint32_t lo = c0 + 2 * t < a.W ? (uint32_t)__ldg(car + c0 + 2 * t) : kNoRow;
                const uint32_t hi = c0 + 2 * t + 1 < a.W ? (uint32_t)__ldg(car + c0 + 2 * t + 1) : kNoRow;
                w[t] = lo | (hi << 16);
            }
        }
    };

    // ---- monotone chain over the window ----
    int n = 0;
    bool overflow = false;
    int tk = 0, tH = 0, sk = 0, sH = 0;  // top and second entries
    for (int c0 = k0; c0 < k1; c0 += 32) {
        uint32_t w[16];
        load32(c0, w);
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            const uint32_t r = (w[t >> 1] >> (16 * (t & 1))) & 0xffffu;
            const int k = c0 + t;
            if (r == kNoRow || k >= k1 || overflow) continue;
            const int d = side ? (int)r - line : line - (int)r;
            const int H = d * d + k * k;
            while (n >= 2 && above_seg(sk, sH, tk, tH, k, H)) {
                --n;
                tk = sk;
                tH = sH;
                if (n >= 2) {
                    sk = k0 + sm.c[n - 2][lane];
                    sH = sm.h[n - 2][lane];
                }
            }
            if (n == kHullCap) {
                overflow = true;
                continue;
            }
            sm.h[n][lane] = H;
            sm.c[n][lane] = (uint16_t)(k - k0);
            ++n;
            sk = tk;
            sH = tH;
            tk = k;
            tH = H;
        }
    }
    sm.lo[lane] = 0;
    sm.hi[lane] = overflow ? 0 : n;
    __syncwarp();

    // ---- bridge merges: groups of g windows, leaders at multiples of 2g ----
    for (int g = 1; g < 32; g <<= 1) {
        if ((lane & (2 * g - 1)) == 0) {
            const int lead = lane, mid = lane + g, end = lane + 2 * g;
            int wa = -1, ia = 0, wb = -1, ib = 0;
            for (int l = mid - 1; l >= lead; --l)
                if (sm.hi[l] > sm.lo[l]) { wa = l; ia = sm.hi[l] - 1; break; }
            for (int l = mid; l < end; ++l)
                if (sm.hi[l] > sm.lo[l]) { wb = l; ib = sm.lo[l]; break; }
            if (wa >= 0 && wb >= 0) {
                int ka = wa * WIN + sm.c[ia][wa], Ha = sm.h[ia][wa];
                int kb = wb * WIN + sm.c[ib][wb], Hb = sm.h[ib][wb];
                for (;;) {
                    bool moved = false;
                    for (;;) {  // the predecessor of a in the left group
                        int wp = wa, ip = ia - 1;
                        if (ip < sm.lo[wp]) {
                            for (wp = wa - 1; wp >= lead && sm.hi[wp] <= sm.lo[wp]; --wp) {}
                            if (wp < lead) break;
                            ip = sm.hi[wp] - 1;
                        }
                        const int kp = wp * WIN + sm.c[ip][wp], Hp = sm.h[ip][wp];
                        if (!above_seg(kp, Hp, ka, Ha, kb, Hb)) break;
                        sm.hi[wa] = ia;  // a is the left group's last vertex
                        wa = wp; ia = ip; ka = kp; Ha = Hp;
                        moved = true;
                    }
                    for (;;) {  // the successor of b in the right group
                        int ws = wb, is = ib + 1;
                        if (is >= sm.hi[ws]) {
                            for (ws = wb + 1; ws < end && sm.hi[ws] <= sm.lo[ws]; ++ws) {}
                            if (ws >= end) break;
                            is = sm.lo[ws];
                        }
                        const int ks = ws * WIN + sm.c[is][ws], Hs = sm.h[is][ws];
                        if (!above_seg(ka, Ha, kb, Hb, ks, Hs)) break;
                        sm.lo[wb] = ib + 1;  // b is the right group's first vertex
                        wb = ws; ib = is; kb = ks; Hb = Hs;
                        moved = true;
                    }
                    if (!moved) break;
                }
            }
        }
        __syncwarp();
    }

    // ---- the window's candidate words (side 0 adds the band's object columns) ----
    const int s = p / a.n_img, im = p - s * a.n_img;
    const int pol = a.pol0 + s;
    const int nrows = min(32, a.Hg - 32 * gb);
    const uint32_t valid = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
    const uint32_t* mrow = a.bmask + ((int64_t)im * a.nb + b) * a.Wp;
    uint32_t* out = a.cand + (((int64_t)p * a.nb + b) * 2 + side) * a.Ww;
    int idx = sm.lo[lane];
    const int ihi = sm.hi[lane];
    for (int c0 = k0; c0 < k1; c0 += 32) {
        uint32_t z = 0;
        while (idx < ihi && k0 + sm.c[idx][lane] < c0 + 32) {
            z |= 1u << ((k0 + sm.c[idx][lane]) & 31);
            ++idx;
        }
        if (overflow) {  // every valid column of the window
            uint32_t w[16];
            load32(c0, w);
#pragma unroll
            for (int t = 0; t < 32; ++t)
                z |= (uint32_t)(((w[t >> 1] >> (16 * (t & 1))) & 0xffffu) != kNoRow) << t;
        }
        if (side == 0) {
            if (c0 + 32 <= a.Wp) {
                const uint4* q = reinterpret_cast<const uint4*>(mrow + c0);
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    const uint4 x = __ldg(q + v);
                    z |= (uint32_t)(pol_mask(x.x, pol, valid) != 0u) << (4 * v);
                    z |= (uint32_t)(pol_mask(x.y, pol, valid) != 0u) << (4 * v + 1);
                    z |= (uint32_t)(pol_mask(x.z, pol, valid) != 0u) << (4 * v + 2);
                    z |= (uint32_t)(pol_mask(x.w, pol, valid) != 0u) << (4 * v + 3);
                }
            } else {
                for (int c = 0; c < 32 && c0 + c < a.Wp; ++c)
                    z |= (uint32_t)(pol_mask(__ldg(mrow + c0 + c), pol, valid) != 0u) << c;
            }
        }
        if (k1 - c0 < 32) z &= (1u << (k1 - c0)) - 1u;  // columns past the row end
        out[c0 >> 5] = z;
    }
}

// ------------------------------------------------------------ per-row stacks
struct BandSmem {
    uint32_t ks[kBandCap][32];   // ring: column | start << 16
    uint16_t rr[kBandCap][32];   // ring: the column's nearest object row
    uint16_t cols[1024];         // candidate columns of one 32-word group
};

template <bool TAKE_NEW>
__global__ void __launch_bounds__(32 * kBandWarps) k_band_rows(BandArgs a) {
    __shared__ BandSmem smem[kBandWarps];
    BandSmem& sm = smem[threadIdx.x >> 5];
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int MASK = kBandCap - 1;
    const int lane = threadIdx.x & 31;
    const int64_t task = (int64_t)blockIdx.x * kBandWarps + (threadIdx.x >> 5);
    if (task >= (int64_t)a.nplanes * a.nb) return;
    const int p = (int)(task / a.nb), b = (int)(task - (int64_t)p * a.nb);
    if (!band_plane(a, p)) return;  // warp-uniform
    const int s = p / a.n_img, im = p - s * a.n_img;
    const int pol = a.pol0 + s;
    const int gb = a.band0 + b;  // global band; rows of the image [32 gb, 32 gb + nrows)
    const int nrows = min(32, a.Hg - 32 * gb);
    const uint32_t valid = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
    const bool active = lane < nrows;
    const uint32_t i = (uint32_t)(32 * gb + lane);  // global row
    const uint32_t upmask = 0xffffffffu >> (31 - lane);
    const int64_t row = (int64_t)p * a.H + 32 * b + lane;  // local row
    uint32_t* gE = a.ent + (active ? row * a.Ws : 0);
    uint16_t* gR = a.entr + (active ? row * a.Ws : 0);
    const uint32_t* cA = a.cand + ((int64_t)p * a.nb + b) * 2 * a.Ww;
    const uint32_t* cB = cA + a.Ww;
    const uint32_t* mrow = a.bmask + ((int64_t)im * a.nb + b) * a.Wp;
    const uint16_t* arow = a.above + ((int64_t)p * a.nb + b) * a.Wp;
    const uint16_t* brow = a.below + ((int64_t)p * a.nb + b) * a.Wp;
    const int W = a.W;

    int n = 0, head = 0, ng = 0;  // ring entries head .. head+n-1; ng entries in the global list
    int tk = 0, ts = 0;           // top entry
    uint32_t tg = 0;

    auto cand = [&](int m, uint32_t r) {
        const uint32_t av = i > r ? i - r : r - i;
        const uint32_t gm = av * av;
        int start = 0;
        for (;;) {
            if (n == 0) {
                if (ng == 0) break;  // empty stack: push with start 0
                --ng;                // reload the list's last entry as the ring's only one
                const uint32_t e = gE[ng];
                const uint16_t rk = gR[ng];
                head = 0;
                sm.ks[0][lane] = e;
                sm.rr[0][lane] = rk;
                n = 1;
                tk = (int)(e & 0xffffu);
                ts = (int)(e >> 16);
                const uint32_t ak = i > rk ? i - rk : rk - i;
                tg = ak * ak;
            }
            // num = g_m - g_k + m^2 - k^2, |num| < 2^31; ts*den, (W-1)*den < 2^31
            const int dm = m - tk;
            const int num = (int)gm - (int)tg + dm * (m + tk);
            const int den = 2 * dm;
            const int lim = ts * den;  // start <= js[idx]: pop (:214)
            if (TAKE_NEW ? num <= lim : num < lim) {
                if (--n > 0) {
                    const int idx = (head + n - 1) & MASK;
                    const uint32_t e = sm.ks[idx][lane];
                    tk = (int)(e & 0xffffu);
                    ts = (int)(e >> 16);
                    const uint32_t rk = sm.rr[idx][lane];
                    const uint32_t ak = i > rk ? i - rk : rk - i;
                    tg = ak * ak;
                }
                continue;
            }
            // push iff start <= W-1 (:218); 0 <= num, quotient < W <= 2^15
            if (TAKE_NEW ? num > (W - 1) * den : num >= (W - 1) * den) return;
            const uint32_t q = small_udiv((uint32_t)num, (uint32_t)den);
            // keep_old: floor(x)+1 ; take_new: ceil(x)   (:205)
            start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * (uint32_t)den)) : (int)q + 1;
            break;
        }
        if (n == kBandCap) {  // full ring: its bottom entry moves to the list
            gE[ng] = sm.ks[head][lane];
            gR[ng] = sm.rr[head][lane];
            ++ng;
            head = (head + 1) & MASK;
            --n;
        }
        const int idx = (head + n) & MASK;
        sm.ks[idx][lane] = (uint32_t)m | ((uint32_t)start << 16);
        sm.rr[idx][lane] = (uint16_t)r;
        ++n;
        tk = m;
        ts = start;
        tg = gm;
    };

    // ---- the band's candidates, 32 mask words (<= 1024 columns) at a time ----
    for (int w0 = 0; w0 < a.Ww; w0 += 32) {
        const int w = w0 + lane;
        const uint32_t cw = w < a.Ww ? (__ldg(cA + w) | __ldg(cB + w)) : 0u;
        const int c = __popc(cw);
        int pre = c;  // inclusive prefix
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, pre, o);
            if (lane >= o) pre += v;
        }
        const int T = __shfl_sync(FULL, pre, 31);
        int pos = pre - c;
        for (uint32_t x = cw; x; x &= x - 1) sm.cols[pos++] = (uint16_t)(32 * w + __ffs(x) - 1);
        __syncwarp();
        for (int t0 = 0; t0 < T; t0 += 32) {
            // lane loads candidate t0 + lane: column, band mask, both carries
            uint32_t kk = 0, mm = 0, cc = 0;
            if (t0 + lane < T) {
                kk = sm.cols[t0 + lane];
                mm = __ldg(mrow + kk);
                cc = (uint32_t)__ldg(arow + kk) | ((uint32_t)__ldg(brow + kk) << 16);
            }
            const int nu = min(32, T - t0);
            for (int u = 0; u < nu; ++u) {
                const int m = (int)__shfl_sync(FULL, kk, u);
                const uint32_t mk = pol_mask(__shfl_sync(FULL, mm, u), pol, valid);
                const uint32_t c2 = __shfl_sync(FULL, cc, u);
                if (!active) continue;
                const uint32_t up = mk & upmask, dn = mk >> lane;
                const uint32_t ra = up ? (uint32_t)(32 * gb + 31 - __clz(up)) : (c2 & 0xffffu);
                const uint32_t rb = dn ? (uint32_t)(i + __ffs(dn) - 1) : (c2 >> 16);
                const uint32_t r = pick_nearest(i, ra, rb);
                if (r != kNoRow) cand(m, r);
            }
        }
        __syncwarp();
    }
    if (!active) return;
    // ---- the final stack is the row's owner list ----
    for (int e = 0; e < n; ++e) {
        const int idx = (head + e) & MASK;
        gE[ng] = sm.ks[idx][lane];
        gR[ng] = sm.rr[idx][lane];
        ++ng;
    }
    if (ng == 0) {  // featureless plane: one "no owner" entry
        gE[0] = kLrInfK;
        gR[0] = kNoRow;
        ng = 1;
    }
    a.nent[row] = ng;
}

// ------------------------------------------------------------------- fill
struct FillSmem {
    uint32_t e[kFillCap];
    uint16_t r[kFillCap];
};

__global__ void __launch_bounds__(32 * kFillWarps) k_rows_fill(RowArgs ra, BandArgs a) {
    extern __shared__ uint4 fill_raw[];
    FillSmem& sm = reinterpret_cast<FillSmem*>(fill_raw)[threadIdx.x >> 5];
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int W = a.W;
    const int64_t total = (int64_t)a.nplanes * a.H;
    const int64_t nw = (int64_t)gridDim.x * kFillWarps;
    const uint32_t sE_addr = (uint32_t)__cvta_generic_to_shared(sm.e);
    const uint32_t sR_addr = (uint32_t)__cvta_generic_to_shared(sm.r);
    const bool donly = ra.D && !ra.S && !ra.LB && !ra.NC;
    for (int64_t row = (int64_t)blockIdx.x * kFillWarps + (threadIdx.x >> 5); row < total; row += nw) {
        const int p = (int)(row / a.H);
        if (!band_plane(a, p)) continue;  // warp-uniform
        const int64_t iR = row - (int64_t)p * a.H;
        const uint32_t gi = (uint32_t)(iR + 32 * a.band0);  // global row
        const int nE = __ldcg(a.nent + row);
        const uint32_t* gE = a.ent + row * a.Ws;
        const uint16_t* gR = a.entr + row * a.Ws;
        int32_t* Drow = ra.D ? reinterpret_cast<int32_t*>(ra.D + p * ra.sD) + iR * W : nullptr;
        float* Srow = ra.S ? reinterpret_cast<float*>(ra.S + p * ra.sS) + iR * W : nullptr;
        int32_t* Lrow = ra.LB ? reinterpret_cast<int32_t*>(ra.LB + p * ra.sL) + iR * W : nullptr;
        int32_t* Nrow = ra.NC ? reinterpret_cast<int32_t*>(ra.NC + p * ra.sN) + iR * W : nullptr;
        if (nE <= kFillCap) {
            __syncwarp();
            for (int q = lane; 4 * q < nE; q += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sE_addr + 16u * q), "l"(gE + 4 * q));
            for (int q = lane; 8 * q < nE; q += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sR_addr + 16u * q), "l"(gR + 8 * q));
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncwarp();
            if (donly)
                lr_fill_row<true>(ra, sm.e, sm.r, nE, gi, Drow, Srow, Lrow, Nrow, 0, W, lane);
            else
                lr_fill_row<false>(ra, sm.e, sm.r, nE, gi, Drow, Srow, Lrow, Nrow, 0, W, lane);
            continue;
        }
        // a long list (dense stretches): 32-column blocks straight from L2
        int base = 0;
        for (int b = 0; b < W; b += 32) {
            const int idx = base + lane;
            const uint32_t we = idx < nE ? __ldcg(gE + idx) : FULL;
            const uint32_t wr = idx < nE ? (uint32_t)__ldcg(gR + idx) : kNoRow;
            const int s = (int)(we >> 16);
            const bool in = lane >= 1 && s <= b + 31;
            const uint32_t Z = __reduce_or_sync(FULL, in ? 1u << (s - b) : 0u);
            const int ow = __popc(Z & ((2u << lane) - 1u));
            const uint32_t ke = __shfl_sync(FULL, we, ow);
            const uint32_t kr = __shfl_sync(FULL, wr, ow);
            const int j = b + lane;
            if (j < W) {
                const uint32_t k = ke & 0xffffu;
                const bool inf = k == kLrInfK;
                const uint32_t av = gi > kr ? gi - kr : kr - gi;
                const int dj = j - (int)k;
                const uint32_t d = inf ? (uint32_t)DFC_INF_I32 : av * av + (uint32_t)(dj * dj);
                if (Drow) __stcs(Drow + j, (int32_t)d);
                if (Srow) __stcs(Srow + j, dist_f32(d));
                if (Lrow) __stcs(Lrow + j, inf ? -1 : (int32_t)(kr * (uint32_t)W + k));
                if (Nrow) __stcs(Nrow + j, inf ? -1 : (int32_t)k);
            }
            const uint32_t s32 = (lane == 0 && base + 32 < nE) ? (__ldcg(gE + base + 32) >> 16) : 0xffffu;
            base += __popc(__ballot_sync(FULL, lane >= 1 && s <= b + 32)) +
                    ((int)__shfl_sync(FULL, s32, 0) <= b + 32 ? 1 : 0);
        }
    }
}

inline int fill_smem_bytes() { return kFillWarps * (int)sizeof(FillSmem); }

}  // namespace dfc
