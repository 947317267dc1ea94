// k_rows_zs.cu -- stage 2 fast path for DENSE rows: zero-split envelopes.
//
// A column z whose pixel (i, z) is itself an object of the transform's
// polarity has g_z = 0.  For any column j > z, (j-z)^2 < (j-k)^2 for every
// k < z, so no parabola left of z can own (or tie) a column right of z, and
// symmetrically.  The zero columns therefore split the row into independent
// gaps: on (z1, z2) the lower envelope only involves the parabolas of columns
// z1..z2, and running the reference stack algorithm (exact_edt.cpp:208-223,
// same tie policy) on those columns gives exactly the reference's owners.
// The left zero z1 is the permanent base of its gap's stack (a later
// parabola m starts beating it at floor((g_m + m^2 - z1^2) / 2(m-z1)) + 1 >
// z1, so it is never popped); it is kept implicit, so a gap's stored entries
// fit in [z1+1, z2] and gaps never overlap in the shared stack array.
//
// One CTA per row: stage the row's nearest rows, block scans give every
// column its enclosing zeros, one thread per gap runs the stack algorithm,
// then every thread fills its own contiguous chunk with 16-byte stores (zero
// columns: D = 0, label = the pixel itself).  Dense polarities (the inside
// of config 2's discs) have short gaps; a row with a gap longer than kZsGap
// is appended to the fallback list and recomputed by k_rows.
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kZsThreads = 256;
constexpr int kZsGap = 256;   // longest gap (columns strictly between zeros) handled here

template <bool TAKE_NEW>
__global__ void __launch_bounds__(kZsThreads) k_rows_zs(RowArgs a, int* fail_rows, int* fail_count) {
    extern __shared__ uint32_t zsm[];
    const int W = a.W;
    const int64_t row = blockIdx.x;
    if (row >= a.total_rows) return;
    const int img = (int)(row / a.H);
    // sparse plane (objects of this polarity <= half the pixels): gaps are long,
    // hand the row straight to the segment kernel
    if ((uint64_t)a.dens[img] * 2 <= (uint64_t)a.H * (uint64_t)a.W) {
        if (threadIdx.x == 0) fail_rows[atomicAdd(fail_count, 1)] = (int)row;
        return;
    }
    const uint32_t i = (uint32_t)(row - (int64_t)img * a.H);
    const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;  // zero column <=> nr == gi
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int per = (W + kZsThreads - 1) / kZsThreads;
    const int c0 = min(t * per, W), c1 = min(c0 + per, W);

    uint16_t* nrs = reinterpret_cast<uint16_t*>(zsm);             // [W (+pad)]
    uint32_t* stk = zsm + ((W + 8) >> 1);                         // [W] gap stacks at z1+1..
    uint16_t* gcnt = reinterpret_cast<uint16_t*>(stk + W);        // [W+1] entries of the gap after z
    int* wlast = reinterpret_cast<int*>(gcnt + ((W + 8) & ~7));   // [8] per-warp scans
    int* wfirst = wlast + 8;
    int* flag = wfirst + 8;

    const uint16_t* rowp = a.nr + img * a.nr_img_stride + (int64_t)i * a.Wp;
    for (int q = t; q < (W + 1) >> 1; q += kZsThreads)
        reinterpret_cast<uint32_t*>(nrs)[q] = __ldg(reinterpret_cast<const uint32_t*>(rowp) + q);
    if (t == 0) *flag = 0;
    __syncthreads();

    // ---- enclosing zeros: exclusive prefix max of the last zero per chunk,
    // exclusive suffix min of the first zero per chunk ----
    int zf = W, zl = -1;
    for (int j = c0; j < c1; ++j)
        if (nrs[j] == gi) {
            if (zf == W) zf = j;
            zl = j;
        }
    int pmax = zl, smin = zf;
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, pmax, o);
        const int d = __shfl_down_sync(0xffffffffu, smin, o);
        if (lane >= o) pmax = max(pmax, u);
        if (lane + o < 32) smin = min(smin, d);
    }
    if (lane == 31) wlast[warp] = pmax;
    if (lane == 0) wfirst[warp] = smin;
    __syncthreads();
    int before = __shfl_up_sync(0xffffffffu, pmax, 1);
    int after = __shfl_down_sync(0xffffffffu, smin, 1);
    if (lane == 0) before = -1;
    if (lane == 31) after = W;
    for (int w = 0; w < warp; ++w) before = max(before, wlast[w]);
    for (int w = warp + 1; w < kZsThreads / 32; ++w) after = min(after, wfirst[w]);
    // before: last zero < c0 (-1 if none); after: first zero >= c1 (W if none)

    // ---- every gap must be short: checked where it ends (a zero, or the row end) ----
    {
        bool bad = false;
        int prev = before;
        for (int j = c0; j < c1; ++j)
            if (nrs[j] == gi) {
                if (j - prev - 1 > kZsGap) bad = true;
                prev = j;
            }
        if (c1 == W && W - prev - 1 > kZsGap) bad = true;
        if (bad) *flag = 1;
    }
    if (__syncthreads_or(*flag)) {
        if (t == 0) fail_rows[atomicAdd(fail_count, 1)] = (int)row;
        return;
    }

    // ---- one thread per gap (the thread holding its first column): the
    // reference stack algorithm on columns z1..z2 with z1 an implicit base ----
    auto gap_scan = [&](int z1, int z2) {  // zeros z1 < z2; -1 / W at the row borders
        const int hi = min(z2, W - 1);     // last column of the domain
        uint32_t* st = stk + (z1 + 1);
        int n = 0;
        int tk = z1, ts = max(z1, 0), tg = 0;  // top = the implicit base while n == 0
        const bool base = z1 >= 0;
        for (int m = z1 + 1; m <= hi; ++m) {
            const uint32_t r = nrs[m];
            if (r == kNoRow) continue;
            const int am = (int)(gi > r ? gi - r : r - gi);
            const int gm = am * am;
            int start = base ? -1 : 0;  // no base, empty stack: owns from column 0
            while (n > 0 || base) {
                // num = v_m - v_k - k^2 + m^2 fits int32; ts*den < 2^32
                const int num = gm - tg + (m * m - tk * tk);
                const uint32_t den = 2u * (uint32_t)(m - tk);
                if (n > 0) {
                    const uint32_t lim = (uint32_t)ts * den;
                    if (num < 0 || (TAKE_NEW ? (uint32_t)num <= lim : (uint32_t)num < lim)) {
                        if (--n > 0) {
                            const uint32_t e = st[n - 1];
                            tk = (int)(e & 0xffffu);
                            ts = (int)(e >> 16);
                            const uint32_t rk = nrs[tk];
                            const int ak = (int)(gi > rk ? gi - rk : rk - gi);
                            tg = ak * ak;
                        } else {
                            tk = z1; ts = max(z1, 0); tg = 0;
                        }
                        continue;
                    }
                }
                // push iff start <= hi; num >= 0 (never pops the base, see above)
                const uint32_t lim2 = (uint32_t)(hi) * den;
                start = (TAKE_NEW ? (uint32_t)num > lim2 : (uint32_t)num >= lim2) ? -2 : 0;
                if (start == 0) {
                    const uint32_t q = small_udiv((uint32_t)num, den);
                    start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * den)) : (int)q + 1;
                }
                break;
            }
            if (start == -2) continue;
            if (start < 0) start = 0;
            st[n++] = (uint32_t)m | ((uint32_t)start << 16);
            tk = m;
            ts = start;
            tg = gm;
        }
        gcnt[z1 + 1] = (uint16_t)n;
    };
    {
        int prev = before;
        for (int j = c0; j < c1; ++j)
            if (nrs[j] == gi) {
                if (j > prev + 1 && prev + 1 >= c0) gap_scan(prev, j);
                prev = j;
            }
        if (prev + 1 < c1 && prev + 1 >= c0) gap_scan(prev, after);  // runs past the chunk
    }
    __syncthreads();

    // ---- fill this thread's chunk ----
    int32_t* Drow = a.D ? reinterpret_cast<int32_t*>(a.D + img * a.sD) + (int64_t)i * W : nullptr;
    float* Srow = a.S ? reinterpret_cast<float*>(a.S + img * a.sS) + (int64_t)i * W : nullptr;
    int32_t* Lrow = a.LB ? reinterpret_cast<int32_t*>(a.LB + img * a.sL) + (int64_t)i * W : nullptr;
    int32_t* Nrow = a.NC ? reinterpret_cast<int32_t*>(a.NC + img * a.sN) + (int64_t)i * W : nullptr;
    int z1 = before;           // zero at or before the current column
    bool in_gap = false;
    const uint32_t* st = nullptr;
    int e = -1, n = 0;         // e = -1: the implicit base (column z1) owns
    uint32_t k = 0, rr = 0, gk = 0;
    int next_start = W;
    auto load = [&]() {
        if (e >= n) {  // no finite parabola at all (featureless short row)
            k = 0;
            rr = kNoRow;
            gk = kInfU;
            next_start = W;
            return;
        }
        if (e < 0) {
            k = (uint32_t)z1;
            rr = gi;
            gk = 0;
        } else {
            const uint32_t ent = st[e];
            k = ent & 0xffffu;
            rr = nrs[k];
            const uint32_t av = gi > rr ? gi - rr : rr - gi;
            gk = av * av;
        }
        next_start = e + 1 < n ? (int)(st[e + 1] >> 16) : W;
    };
    auto cell = [&](int j, int32_t& d, uint32_t& kk, uint32_t& rk) {
        if (nrs[j] == gi) {  // zero column: the pixel itself
            z1 = j;
            in_gap = false;
            d = 0;
            kk = (uint32_t)j;
            rk = gi;
            return;
        }
        if (!in_gap) {
            in_gap = true;
            st = stk + (z1 + 1);
            n = gcnt[z1 + 1];
            e = z1 >= 0 ? -1 : 0;  // base owns until the first entry's start
            while (e + 1 < n && (int)(st[e + 1] >> 16) <= j) ++e;
            load();
        }
        while (j >= next_start) {
            ++e;
            load();
        }
        const int dj = j - (int)k;
        d = gk == kInfU ? DFC_INF_I32 : (int32_t)(gk + (uint32_t)(dj * dj));
        kk = k;
        rk = rr;
    };
    auto lab_of = [&](uint32_t kk, uint32_t rk) -> int32_t {
        return rk == kNoRow ? -1 : (int32_t)(rk * (uint32_t)W + kk);
    };
    if (a.vec && (per & 3) == 0) {
        for (int j = c0; j < c1; j += 4) {
            int4 d4;
            uint32_t k0, k1, k2, k3, r0, r1, r2, r3;
            cell(j, d4.x, k0, r0);
            cell(j + 1, d4.y, k1, r1);
            cell(j + 2, d4.z, k2, r2);
            cell(j + 3, d4.w, k3, r3);
            if (Drow) __stcs(reinterpret_cast<int4*>(Drow + j), d4);
            if (Srow)
                __stcs(reinterpret_cast<float4*>(Srow + j),
                       make_float4(dist_f32(d4.x), dist_f32(d4.y), dist_f32(d4.z), dist_f32(d4.w)));
            if (Lrow)
                __stcs(reinterpret_cast<int4*>(Lrow + j),
                       make_int4(lab_of(k0, r0), lab_of(k1, r1), lab_of(k2, r2), lab_of(k3, r3)));
            if (Nrow)
                __stcs(reinterpret_cast<int4*>(Nrow + j),
                       make_int4(r0 == kNoRow ? -1 : (int)k0, r1 == kNoRow ? -1 : (int)k1,
                                 r2 == kNoRow ? -1 : (int)k2, r3 == kNoRow ? -1 : (int)k3));
        }
    } else {
        for (int j = c0; j < c1; ++j) {
            int32_t d;
            uint32_t kk, rk;
            cell(j, d, kk, rk);
            if (Drow) Drow[j] = d;
            if (Srow) Srow[j] = dist_f32((uint32_t)d);
            if (Lrow) Lrow[j] = lab_of(kk, rk);
            if (Nrow) Nrow[j] = rk == kNoRow ? -1 : (int32_t)kk;
        }
    }
}

template <bool TAKE_NEW>
inline const void* zs_kernel_ptr() {
    return (const void*)k_rows_zs<TAKE_NEW>;
}

inline int zs_smem_bytes(int W) { return (((W + 8) >> 1) + W + (((W + 8) & ~7) >> 1) + 17) * 4; }

}  // namespace dfc
