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
//              is exact (the row pass evaluates each candidate's true g_k(i)).
//  k_hull      one CTA prunes one compact point list towards its lower hull
//              (data-parallel rounds: a point above the chord of two list
//              neighbours goes, survivors are compacted); filters at coarse
//              lines over all columns (per window, then per line), at the
//              groups' lines over the coarse filter plus the object columns
//              in between (see "hull filter" below).  Output: candidate bit
//              masks [plane][group][side][W/32].
//  k_band_rows_fill  CTA = (plane, band), 8 warps.
//              Stack phase (band_rows_body): warp = one of 8 column chunks of
//              equal candidate counts, lane = row: the reference's stack
//              algorithm over the chunk's candidates only (g from the band mask
//              and the carries, the upper row on ties, exact_edt.cpp:351), the
//              top kBandCap entries in a shared-memory ring that spills its
//              bottom to the row's list in global memory and reloads from it --
//              the stack is unbounded, no row needs a fallback.  The final
//              stack is the row's owner list (column | start << 16, nearest row).
//              Fill phase (band_fill_body): warp = 4 of the band's rows, the
//              rows' lists staged by TMA bulk copies (two buffers, mbarriers),
//              then the shared lr_fill_row (k_rows_lr.cu): lane = column,
//              16-byte streaming stores -- the HBM-bound part (C5: 4 B/px).
//
// tests/band_model.py is the statement-level model (fuzzed against brute
// force for both tie rules with small windows, lanes and ring capacities).
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kBandWarps = 8;       // k_band_rows: warps (column chunks) per band
constexpr int kBandCap = 16;        // ring entries per lane (power of two)
constexpr int kCandCap = 2048;      // candidates of a band listed in shared memory
constexpr int kFillCap = 512;       // list entries staged per warp and buffer (the fill phase); a chunk of a listed
                                    // band holds ~kCandCap / kBandWarps candidates

struct BandArgs {
    const uint32_t* bmask;   // [img][nb][Wp] bit r = row 32 b + r nonzero
    const uint16_t* above;   // [plane][nb][Wp] nearest object row above the band (kNoRow: none)
    const uint16_t* below;   // [plane][nb][Wp] nearest object row below the band
    uint32_t* cand;          // [plane][group][2][Ww] candidate columns (side 0: above + the group's bands)
    const unsigned long long* counts;  // object pixels per plane
    uint32_t* ent;           // per row list: column | start << 16, at row * Ws
    uint16_t* entr;          // the entries' nearest object rows
    int* nent;               // entries per (row, chunk)
    int* cbound;             // per (plane, band): the chunks' first columns, then W
    int64_t Ws;              // list stride per row (entries)
    int H, W, Wp, nb, Ww, n_img, pol0, nplanes;
    // row stripes (the sharded path): local band b is global band band0 + b of
    // an image of Hg rows; plane p's local rows are [0, H).  Single images:
    // band0 = 0, Hg = H.
    int band0, Hg;
    int group, ngroups;      // bands per candidate group (k_hull<2>), groups per plane
    uint32_t* objcol = nullptr;  // [plane][nb][Ww] columns with an object in the band (null: built from bmask)
    uint32_t* objpre;        // ... OR'ed over the bands from the start of the band's 32 (in its coarse group)
    uint32_t* objsuf;        // ... OR'ed over the bands to the end of the band's 32
    uint32_t* coarse;        // [plane][ncoarse][2][Ww] hulls at the coarse groups' first / last lines
    int cbands, ncoarse;     // bands per coarse group (a multiple of group), coarse groups per plane
    bool pts_gate;           // point planes belong to k_rows_pts
    bool all_planes;         // every plane (the sharded path), not only the sparse ones
};

// The planes this path owns: sparse, not a point plane.
__device__ __forceinline__ bool band_plane(const BandArgs& a, int p) {
    return a.all_planes || (lr_plane(a.counts, p, a.Hg, a.W) && !pts_plane(a.counts, p, a.pts_gate));
}

// ---------------------------------------------------------------- hull filter
// Bands come in groups of G (a.group), groups in coarse groups of a.cbands
// bands.  For band b of group [gb0, gb1] inside coarse group [cb0, cb1]:
//   A-candidates(b) <= hullA(line 32 gb0) + {columns with an object in bands gb0 .. b-1}
//   hullA(line 32 gb0) <= hullA(line 32 cb0) + {columns with an object in bands cb0 .. gb0-1}
// because an object above an earlier line whose cell (among the objects above
// the later line) crosses the later line also crosses the earlier one
// (convexity, the same argument as above); symmetrically below with the last
// bands.  The hull of a point set that contains every hull point IS the hull,
// so only the coarse lines see all W columns; a group line sees the coarse
// hull plus the object columns in between (C5: ~10^3 points, not 32768).
//
// One CTA filters one compact point list in shared memory (column, H = d^2 +
// k^2 < 2^31) by cta_prune below: rounds of "a point strictly above the chord
// of two list neighbours goes", survivors compacted in place.  The result is a
// superset of the lower hull with collinear points kept (ties), which is all
// the argument above needs -- a group line's list must CONTAIN the coarse
// line's hull points, and the candidates must CONTAIN the group line's.
//   K1a / k_band_objcols  object-column bits per band; k_objcol_runs their
//                   running ORs over runs of 32 bands
//   k_hull<0>       CTA = (plane, coarse group, side, window of 1024 columns):
//                   the window's filter over every column with a carry
//   k_hull<1>       CTA = (plane, coarse group, side): the windows' survivors
//                   filtered together
//   k_hull<2>       CTA = (plane, group, side): the coarse line's survivors +
//                   the object columns in between, filtered at the group's
//                   line; side 0 also adds the group's own object columns.
//                   Output: candidate bits [plane][group][side][W/32].
// A list longer than kHullCap is passed through unfiltered (a superset).
constexpr int kHullCap = 2048;     // points per warp (k_hull<1>, k_hull<2>)
constexpr int kHullWinCap = 1024;  // k_hull<0>: a window of 32 words
constexpr int kHullThreads = 256;  // one CTA per line (window)
constexpr int kCoarseBands = 32;   // bands per coarse group (rounded to a multiple of the group)
constexpr int kPruneRounds = 10;

// Object-column bits per band from the band masks (the sharded path, whose
// masks are repacked column tiles; single images get them from K1a).
__global__ void __launch_bounds__(256) k_band_objcols(BandArgs a) {
    constexpr unsigned FULL = 0xffffffffu;
    const int p = blockIdx.z;
    if (!band_plane(a, p)) return;  // CTA-uniform
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = p / a.n_img, im = p - s * a.n_img;
    const int pol = a.pol0 + s;
    for (int b = blockIdx.y; b < a.nb; b += gridDim.y) {
        const int nrows = min(32, a.Hg - 32 * (a.band0 + b));
        const uint32_t valid = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
        const bool on = k < a.W && pol_mask(__ldg(a.bmask + ((int64_t)im * a.nb + b) * a.Wp + k), pol, valid) != 0u;
        const uint32_t word = __ballot_sync(FULL, on);
        if ((threadIdx.x & 31) == 0 && (k >> 5) < a.Ww) a.objcol[((int64_t)p * a.nb + b) * a.Ww + (k >> 5)] = word;
    }
}

// Running ORs of the object-column words inside each run of 32 bands of a
// coarse group: pre[b] = OR over the run's bands up to b, suf[b] = from b on.
// Thread = (word, run of 32 bands), 32 independent loads.
__global__ void __launch_bounds__(128) k_objcol_runs(BandArgs a) {
    const int p = blockIdx.z, cg = blockIdx.y;
    if (!band_plane(a, p)) return;  // CTA-uniform
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= a.Ww) return;
    const int cb0 = cg * a.cbands, cb1 = min(a.nb - 1, cb0 + a.cbands - 1);
    for (int bb = cb0; bb <= cb1; bb += 32) {
        const int nbb = min(32, cb1 - bb + 1);
        const int64_t at = ((int64_t)p * a.nb + bb) * a.Ww + w;
        uint32_t x[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) x[t] = t < nbb ? a.objcol[at + (int64_t)t * a.Ww] : 0u;
        uint32_t run = 0;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
            run |= x[t];
            if (t < nbb) a.objpre[at + (int64_t)t * a.Ww] = run;
        }
        run = 0;
#pragma unroll
        for (int t = 31; t >= 0; --t) {
            run |= x[t];
            if (t < nbb) a.objsuf[at + (int64_t)t * a.Ww] = run;
        }
    }
}

// b strictly above the segment a-c (H differences fit int32, column
// differences < 2^15: one IMAD.WIDE each)
__device__ __forceinline__ bool hull_above(int ka, int Ha, int kb, int Hb, int kc, int Hc) {
    return (long long)(Hb - Ha) * (kc - kb) > (long long)(Hc - Hb) * (kb - ka);
}

// Prune the compact point list c / H [0, n) (ascending columns) towards its
// lower hull, data-parallel over the CTA: in every round point i goes if it
// lies strictly above the chord of its list neighbours i - s and i + s for
// some stride s = 1, 2, .., 64 (a point above a chord of two points of the set
// is no hull point, whatever happens to those two), then the survivors are
// compacted in place (every thread holds its points in registers across the
// barrier).  Any number of rounds leaves a superset of the hull (collinear
// points kept); on C5's lines 5 rounds reach the hull itself (10^4 -> ~10^2
// points, profiles/r02/prune_study.txt).  Thread = points tid + kHullThreads t.
// Returns the new n (CTA-uniform).
template <int CAP>
__device__ __forceinline__ int cta_prune(uint16_t* c, int32_t* H, int* wsum, int n, int tid) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int NT = CAP / kHullThreads;  // points per thread
    constexpr int NW = kHullThreads / 32;
    const int lane = tid & 31, warp = tid >> 5;
    for (int round = 0; round < kPruneRounds && n >= 3; ++round) {
        int ki[NT], Hi[NT];
        uint32_t keep = 0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int i = kHullThreads * t + tid;
            ki[t] = 0;
            Hi[t] = 0;
            if (i < n) {
                ki[t] = c[i];
                Hi[t] = H[i];
                bool ab = false;
#pragma unroll
                for (int s = 1; s <= 64; s <<= 1)
                    if (i >= s && i + s < n) ab |= hull_above(c[i - s], H[i - s], ki[t], Hi[t], c[i + s], H[i + s]);
                keep |= (uint32_t)!ab << t;
            }
        }
        // order-preserving positions: counts per (t, warp), t-major
        uint32_t bal[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            bal[t] = __ballot_sync(FULL, (keep >> t) & 1u);
            if (lane == 0) wsum[t * NW + warp] = __popc(bal[t]);
        }
        __syncthreads();  // every read of this round's list is done; the counts are visible
        int base[NT], total = 0;
        {
            // NT * NW <= 64 counts: every warp scans them with two per lane
            const int e0 = 2 * lane, e1 = 2 * lane + 1;
            const int v0 = e0 < NT * NW ? wsum[e0] : 0, v1 = e1 < NT * NW ? wsum[e1] : 0;
            int incl = v0 + v1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            total = __shfl_sync(FULL, incl, 31);
            const int ex0 = incl - v0 - v1, ex1 = ex0 + v0;  // exclusive prefixes of entries e0, e1
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int e = t * NW + warp;
                const int a0 = __shfl_sync(FULL, ex0, e >> 1), a1 = __shfl_sync(FULL, ex1, e >> 1);
                base[t] = (e & 1) ? a1 : a0;
            }
        }
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if ((keep >> t) & 1u) {
                const int pos = base[t] + __popc(bal[t] & ((1u << lane) - 1u));
                c[pos] = (uint16_t)ki[t];
                H[pos] = Hi[t];
            }
        __syncthreads();
        if (total == n) break;
        n = total;
    }
    return n;
}

// MODE 0: window filters of the coarse lines; 1: the coarse lines' filters
// from their windows' (in place); 2: the group lines' filters.  One CTA per
// line (window).
template <int MODE>
__global__ void __launch_bounds__(kHullThreads) k_hull(BandArgs a) {
    constexpr int CAP = MODE == 0 ? kHullWinCap : kHullCap;
    constexpr int NW = kHullThreads / 32;
    __shared__ int32_t H0[CAP];
    __shared__ uint16_t c0[CAP];
    __shared__ int wsum[64];
    __shared__ int wcnt[NW];
    constexpr unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwin = (a.Ww + 31) / 32;
    const int64_t per_plane = MODE == 0 ? (int64_t)a.ncoarse * 2 * nwin : MODE == 1 ? (int64_t)a.ncoarse * 2
                                                                                    : (int64_t)a.ngroups * 2;
    const int64_t task = blockIdx.x;
    const int p = (int)(task / per_plane);
    if (p >= a.nplanes || !band_plane(a, p)) return;  // CTA-uniform
    int t = (int)(task - (int64_t)p * per_plane);
    int win = 0;
    if (MODE == 0) {
        win = t % nwin;
        t /= nwin;
    }
    const int side = t & 1, grp = t >> 1;  // coarse group (MODE 0, 1) or group (MODE 2)
    if (grp >= (MODE == 2 ? a.ngroups : a.ncoarse)) return;
    const int nb = a.nb;
    const int bper = MODE == 2 ? a.group : a.cbands;
    const int gb0 = grp * bper, gb1 = min(nb - 1, gb0 + bper - 1);
    const int kb = side ? gb1 : gb0;  // the key band of this side
    const int line = side ? min(32 * (a.band0 + kb) + 31, a.Hg - 1) : 32 * (a.band0 + kb);
    const uint16_t* car = (side ? a.below : a.above) + ((int64_t)p * nb + kb) * a.Wp;
    const int w0 = MODE == 0 ? 32 * win : 0, w1 = MODE == 0 ? min(a.Ww, w0 + 32) : a.Ww;
    const int cg = MODE == 2 ? gb0 / a.cbands : grp;
    uint32_t* coarse = a.coarse + (((int64_t)p * a.ncoarse + cg) * 2 + side) * a.Ww;
    uint32_t* out = MODE == 2 ? a.cand + (((int64_t)p * a.ngroups + grp) * 2 + side) * a.Ww : coarse;
    const uint32_t* oc = a.objcol + (int64_t)p * nb * a.Ww;
    // object columns between the coarse line and this group's line
    const int cb0 = cg * a.cbands, cb1 = min(nb - 1, cb0 + a.cbands - 1);
    const int r0 = side ? gb1 + 1 : cb0, r1 = side ? cb1 : gb0 - 1;

    auto in_word = [&](int w) -> uint32_t {  // the input points of word w
        if (MODE == 0) {                     // every column with a carry
            uint32_t x = 0;
            const int c0w = 32 * w;
            if (c0w + 32 <= a.Wp) {
                const uint4* q = reinterpret_cast<const uint4*>(car + c0w);
                uint4 y[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) y[v] = __ldg(q + v);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const uint32_t u[4] = {y[v].x, y[v].y, y[v].z, y[v].w};
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        x |= (uint32_t)((u[z] & 0xffffu) != kNoRow) << (8 * v + 2 * z);
                        x |= (uint32_t)((u[z] >> 16) != kNoRow) << (8 * v + 2 * z + 1);
                    }
                }
            } else {
                for (int c = 0; c < 32 && c0w + c < a.Wp; ++c) x |= (uint32_t)(__ldg(car + c0w + c) != kNoRow) << c;
            }
            if (a.W - c0w < 32) x &= a.W > c0w ? (1u << (a.W - c0w)) - 1u : 0u;
            return x;
        }
        uint32_t x = coarse[w];
        if (MODE == 2) {  // bands r0 .. r1 of the coarse group: running ORs, restarted every 32 bands
            const uint32_t* run = (side ? a.objsuf : a.objpre) + (int64_t)p * nb * a.Ww;
            if (side) {
                x |= __ldg(run + (int64_t)r0 * a.Ww + w);  // r0 .. the end of r0's 32 bands
                for (int b = cb0 + ((r0 - cb0) | 31) + 1; b <= r1; b += 32) x |= __ldg(run + (int64_t)b * a.Ww + w);
            } else {
                x |= __ldg(run + (int64_t)r1 * a.Ww + w);  // the start of r1's 32 bands .. r1
                for (int b = cb0 + ((r1 - cb0) & ~31) - 1; b >= r0; b -= 32) x |= __ldg(run + (int64_t)b * a.Ww + w);
            }
        }
        return x;
    };
    auto base_word = [&](int w) -> uint32_t {  // side 0 of a group: its own object columns
        uint32_t x = 0;
        if (MODE == 2 && side == 0)
            for (int b = gb0; b <= gb1; ++b) x |= __ldg(oc + (int64_t)b * a.Ww + w);
        return x;
    };

    if (MODE == 2 && r1 < r0) {  // the group's line is the coarse line: already filtered
        for (int w = tid; w < a.Ww; w += kHullThreads) out[w] = coarse[w] | base_word(w);
        return;
    }
    // ---- gather the points (compact, ascending columns): thread = a run of
    // consecutive words, all of them loaded before any is used ----
    constexpr int PER = MODE == 0 ? 1 : 4;  // words per thread: 32 (a window) or <= 1024 (W <= 32768)
    const int lw0 = w0 + tid * PER;
    uint32_t x[PER];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        x[u] = lw0 + u < w1 ? in_word(lw0 + u) : 0u;
        cnt += __popc(x[u]);
    }
    int pre = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, pre, o);
        if (lane >= o) pre += v;
    }
    if (lane == 31) wcnt[warp] = pre;
    __syncthreads();
    int pos = pre - cnt, n = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int v = wcnt[w];
        if (w < warp) pos += v;
        n += v;
    }
    if (n > CAP) {  // too many points for one CTA: unfiltered (a superset of the hull)
#pragma unroll
        for (int u = 0; u < PER; ++u)
            if (lw0 + u < w1) out[lw0 + u] = x[u] | base_word(lw0 + u);
        return;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u)
        for (uint32_t y = x[u]; y; y &= y - 1) c0[pos++] = (uint16_t)(32 * (lw0 + u) + __ffs(y) - 1);
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += 4 * kHullThreads) {  // H = d^2 + k^2, four carries in flight
        int cr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kHullThreads + tid;
            cr[u] = i < n ? (int)__ldg(car + c0[i]) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kHullThreads + tid;
            if (i < n) {
                const int k = c0[i];
                const int d = side ? cr[u] - line : line - cr[u];  // a listed column has a carry
                H0[i] = d * d + k * k;
            }
        }
    }
    __syncthreads();
    n = cta_prune<CAP>(c0, H0, wsum, n, tid);
    // ---- the survivors' bits over the base words ----
#pragma unroll
    for (int u = 0; u < PER; ++u)
        if (lw0 + u < w1) out[lw0 + u] = base_word(lw0 + u);
    __syncthreads();
    for (int i = tid; i < n; i += kHullThreads) {
        const int k = c0[i];
        atomicOr(out + (k >> 5), 1u << (k & 31));
    }
}

// ------------------------------------------------------------ per-row stacks
// CTA = (plane, band), kBandWarps warps.  The band's candidates (the group's
// words) are listed in shared memory with their band mask and carries, then
// cut into kBandWarps chunks of equal candidate counts; chunk w covers the
// columns [c0, c1) from its first candidate to the next chunk's.  Lane = row:
// the owners of c0 - 1 and c1 - 1 (exact, by an outward search over the
// candidate list that stops once the nearest unexamined column d has d^2 >
// best) bound the candidates any column of the chunk can take (owners are
// monotone in j under either tie rule, as in k_rows_lr.cu), and the
// reference's stack algorithm runs over that range with the domain restricted
// to [c0, c1): an empty stack pushes with start c0, a parabola starting past
// c1 - 1 is not pushed (:218).  The top kBandCap entries of each stack live
// in a shared-memory ring that spills its bottom to the row's list for the
// chunk (global, at row * Ws + c0: a chunk's stack holds distinct starts in
// [c0, c1), so the lists of a row never overlap) and reloads from it.  Bands
// with more than kCandCap candidates run the whole row in one chunk, with the
// candidates streamed 1024 at a time.
struct BandSmem {
    uint16_t col[kCandCap];      // the band's candidate columns, ascending
    uint32_t msk[kCandCap];      // their band masks (raw: nonzero rows)
    uint32_t car[kCandCap];      // their carries: above | below << 16
    uint32_t ks[kBandWarps][kBandCap][32];  // rings: column | start << 16
    uint16_t rr[kBandWarps][kBandCap][32];  // rings: the column's nearest object row
    int warp_n[kBandWarps + 1];
    int n;
};

// The stacks of band `task` (= plane * nb + band).  Warps leave at different
// points after the last CTA barrier inside; the caller adds its own barrier
// before anything that reads the lists.
template <bool TAKE_NEW>
__device__ __forceinline__ void band_rows_body(const BandArgs& a, BandSmem& sm, int64_t task) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int MASK = kBandCap - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int p = (int)(task / a.nb), b = (int)(task - (int64_t)p * a.nb);
    const int s = p / a.n_img, im = p - s * a.n_img;
    const int pol = a.pol0 + s;
    const int gb = a.band0 + b;  // global band; rows of the image [32 gb, 32 gb + nrows)
    const int nrows = min(32, a.Hg - 32 * gb);
    const uint32_t valid = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
    const bool active = lane < nrows;
    const uint32_t i = (uint32_t)(32 * gb + lane);  // global row
    const uint32_t upmask = 0xffffffffu >> (31 - lane);
    const int64_t row = (int64_t)p * a.H + 32 * b + lane;  // local row
    const uint32_t* cA = a.cand + ((int64_t)p * a.ngroups + b / a.group) * 2 * a.Ww;
    const uint32_t* cB = cA + a.Ww;
    const uint32_t* mrow = a.bmask + ((int64_t)im * a.nb + b) * a.Wp;
    const uint16_t* arow = a.above + ((int64_t)p * a.nb + b) * a.Wp;
    const uint16_t* brow = a.below + ((int64_t)p * a.nb + b) * a.Wp;
    const int W = a.W;
    int* bounds = a.cbound + task * (kBandWarps + 1);

    // ---- 1. the candidate list: a CTA prefix over the words ----
    const int per = (a.Ww + blockDim.x - 1) / blockDim.x;  // words per thread, consecutive
    const int w0 = tid * per, w1 = min(a.Ww, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(__ldg(cA + w) | __ldg(cB + w));
    int pre = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, pre, o);
        if (lane >= o) pre += v;
    }
    if (lane == 31) sm.warp_n[warp + 1] = pre;
    __syncthreads();
    if (tid == 0) {
        sm.warp_n[0] = 0;
        for (int w = 1; w <= kBandWarps; ++w) sm.warp_n[w] += sm.warp_n[w - 1];
        sm.n = sm.warp_n[kBandWarps];
    }
    __syncthreads();
    const int n = sm.n;
    const bool streamed = n > kCandCap;
    if (!streamed) {
        int pos = sm.warp_n[warp] + pre - cnt;
        for (int w = w0; w < w1; ++w)
            for (uint32_t x = __ldg(cA + w) | __ldg(cB + w); x; x &= x - 1) {
                const int k = 32 * w + __ffs(x) - 1;
                sm.col[pos] = (uint16_t)k;
                sm.msk[pos] = __ldg(mrow + k);
                sm.car[pos] = (uint32_t)__ldg(arow + k) | ((uint32_t)__ldg(brow + k) << 16);
                ++pos;
            }
    }
    __syncthreads();
    // chunk w: from the 32-column block of candidate w n / N to the next
    // chunk's (aligned, so the fill's 16-byte stores stay aligned)
    const int NC = streamed ? 1 : kBandWarps;
    if (warp >= NC) return;
    const int ilo = (int)((int64_t)warp * n / NC), ihi = (int)((int64_t)(warp + 1) * n / NC);
    const int c0 = (warp == 0 || streamed || ilo >= n) ? (warp == 0 || streamed ? 0 : W) : (sm.col[ilo] & ~31);
    const int c1 = (warp == NC - 1 || ihi >= n) ? W : (sm.col[ihi] & ~31);
    if (lane == 0) {
        bounds[warp] = c0;
        if (warp == NC - 1)
            for (int w = NC; w <= kBandWarps; ++w) bounds[w] = W;
    }
    if (c0 >= c1) {  // an empty chunk (fewer candidates than chunks)
        if (active) a.nent[row * kBandWarps + warp] = 0;
        return;
    }

    // nearest object row of a candidate column for this lane's row (upper on ties)
    auto nearest = [&](uint32_t m, uint32_t c2) -> uint32_t {
        const uint32_t mk = pol_mask(m, pol, valid);
        const uint32_t up = mk & upmask, dn = mk >> lane;
        const uint32_t ra = up ? (uint32_t)(32 * gb + 31 - __clz(up)) : (c2 & 0xffffu);
        const uint32_t rb = dn ? (uint32_t)(i + __ffs(dn) - 1) : (c2 >> 16);
        return pick_nearest(i, ra, rb);
    };

    uint32_t* gE = a.ent + (active ? row * a.Ws + c0 : 0);
    uint16_t* gR = a.entr + (active ? row * a.Ws + c0 : 0);
    uint32_t (*ks)[32] = sm.ks[warp];
    uint16_t (*rr)[32] = sm.rr[warp];
    int nst = 0, head = 0, ng = 0;  // ring entries head .. head+nst-1; ng entries in the list
    int tk = 0, ts = 0;             // top entry
    uint32_t tg = 0;
    const int cmax = c1 - 1;

    // one candidate column m with nearest row r: pops, then a push (exact_edt.cpp:208-223)
    auto cand = [&](int m, uint32_t r) {
        const uint32_t av = i > r ? i - r : r - i;
        const uint32_t gm = av * av;
        int start = c0;
        for (;;) {
            if (nst == 0) {
                if (ng == 0) break;  // empty stack: push with start c0
                --ng;                // reload the list's last entry as the ring's only one
                const uint32_t e = gE[ng];
                const uint16_t rk = gR[ng];
                head = 0;
                ks[0][lane] = e;
                rr[0][lane] = rk;
                nst = 1;
                tk = (int)(e & 0xffffu);
                ts = (int)(e >> 16);
                const uint32_t ak = i > rk ? i - rk : rk - i;
                tg = ak * ak;
            }
            // num = g_m - g_k + m^2 - k^2, |num| < 2^31; ts*den, cmax*den < 2^31
            const int dm = m - tk;
            const int num = (int)gm - (int)tg + dm * (m + tk);
            const int den = 2 * dm;
            const int lim = ts * den;  // start <= js[idx]: pop (:214)
            if (TAKE_NEW ? num <= lim : num < lim) {
                if (--nst > 0) {
                    const int idx = (head + nst - 1) & MASK;
                    const uint32_t e = ks[idx][lane];
                    tk = (int)(e & 0xffffu);
                    ts = (int)(e >> 16);
                    const uint32_t rk = rr[idx][lane];
                    const uint32_t ak = i > rk ? i - rk : rk - i;
                    tg = ak * ak;
                }
                continue;
            }
            // push iff start <= c1-1 (:218 with cols -> c1); 0 <= num, quotient < W <= 2^15
            if (TAKE_NEW ? num > cmax * den : num >= cmax * den) return;
            const uint32_t q = small_udiv((uint32_t)num, (uint32_t)den);
            // keep_old: floor(x)+1 ; take_new: ceil(x)   (:205)
            start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * (uint32_t)den)) : (int)q + 1;
            break;
        }
        if (nst == kBandCap) {  // full ring: its bottom entry moves to the list
            gE[ng] = ks[head][lane];
            gR[ng] = rr[head][lane];
            ++ng;
            head = (head + 1) & MASK;
            --nst;
        }
        const int idx = (head + nst) & MASK;
        ks[idx][lane] = (uint32_t)m | ((uint32_t)start << 16);
        rr[idx][lane] = (uint16_t)r;
        ++nst;
        tk = m;
        ts = start;
        tg = gm;
    };

    if (!streamed) {
        // ---- 2. exact scan bounds: the owners of c0 - 1 and c1 - 1 ----
        // index of the owner of column x among all candidates (outward search)
        auto owner_idx = [&](int x) -> int {
            int lo = 0, hi = n;  // first candidate >= x (warp-uniform binary search)
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((int)sm.col[mid] < x) lo = mid + 1; else hi = mid;
            }
            uint32_t best = kInfU;
            int bi = -1, bk = 0;
            int l = lo - 1, r = lo;
            bool go = active;
            for (;;) {
                const int dl = l >= 0 ? x - (int)sm.col[l] : INT32_MAX;
                const int dr = r < n ? (int)sm.col[r] - x : INT32_MAX;
                const int d = min(dl, dr);
                go = go && d != INT32_MAX && (uint32_t)d * (uint32_t)d <= best;
                if (!__any_sync(FULL, go)) break;
                const bool left = dl <= dr;  // warp-uniform: same x, same list
                const int t = left ? l : r;
                if (go) {
                    const uint32_t rw = nearest(sm.msk[t], sm.car[t]);
                    if (rw != kNoRow) {
                        const uint32_t av = i > rw ? i - rw : rw - i;
                        const uint32_t v = av * av + (uint32_t)d * (uint32_t)d;
                        const int k = sm.col[t];
                        if (v < best || (v == best && (TAKE_NEW ? k > bk : k < bk))) {
                            best = v;
                            bi = t;
                            bk = k;
                        }
                    }
                }
                if (left) --l; else ++r;
            }
            return bi;
        };
        int iS = 0, iE = n - 1;
        if (c0 > 0) iS = owner_idx(c0 - 1);
        if (c1 < W) iE = owner_idx(c1 - 1);
        // ---- 3. the stack over candidates [iS, iE] (a featureless row: no owner) ----
        const int jS = __reduce_min_sync(FULL, (unsigned)(active && iS >= 0 ? iS : n));
        const int jE = (int)__reduce_max_sync(FULL, (unsigned)(active && iE >= 0 ? iE + 1 : 0)) - 1;
        for (int t = jS; t <= jE; ++t) {
            if (!active || iS < 0 || t < iS || t > iE) continue;
            const uint32_t r = nearest(sm.msk[t], sm.car[t]);
            if (r != kNoRow) cand((int)sm.col[t], r);
        }
    } else {
        // ---- dense band: the whole row, candidates streamed 1024 at a time ----
        uint16_t* cols = sm.col;  // reused as the group's column list
        for (int wg = 0; wg < a.Ww; wg += 32) {
            const int w = wg + lane;
            const uint32_t cw = w < a.Ww ? (__ldg(cA + w) | __ldg(cB + w)) : 0u;
            const int c = __popc(cw);
            int pre2 = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(FULL, pre2, o);
                if (lane >= o) pre2 += v;
            }
            const int T = __shfl_sync(FULL, pre2, 31);
            int pos = pre2 - c;
            for (uint32_t x = cw; x; x &= x - 1) cols[pos++] = (uint16_t)(32 * w + __ffs(x) - 1);
            __syncwarp();
            for (int t0 = 0; t0 < T; t0 += 32) {
                uint32_t kk = 0, mm = 0, cc = 0;
                if (t0 + lane < T) {
                    kk = cols[t0 + lane];
                    mm = __ldg(mrow + kk);
                    cc = (uint32_t)__ldg(arow + kk) | ((uint32_t)__ldg(brow + kk) << 16);
                }
                const int nu = min(32, T - t0);
                for (int u = 0; u < nu; ++u) {
                    const int m = (int)__shfl_sync(FULL, kk, u);
                    const uint32_t m2 = __shfl_sync(FULL, mm, u);
                    const uint32_t c2 = __shfl_sync(FULL, cc, u);
                    if (!active) continue;
                    const uint32_t r = nearest(m2, c2);
                    if (r != kNoRow) cand(m, r);
                }
            }
            __syncwarp();
        }
    }
    if (!active) return;
    // ---- the final stack is the chunk's owner list ----
    for (int e = 0; e < nst; ++e) {
        const int idx = (head + e) & MASK;
        gE[ng] = ks[idx][lane];
        gR[ng] = rr[idx][lane];
        ++ng;
    }
    if (ng == 0) {  // a featureless row: one "no owner" entry
        gE[0] = kLrInfK | ((uint32_t)c0 << 16);
        gR[0] = kNoRow;
        ng = 1;
    }
    a.nent[row * kBandWarps + warp] = ng;
}


// ------------------------------------------------------------------- fill
struct FillSmem {
    uint32_t e[kFillCap];
    uint16_t r[kFillCap];
};

// One row of a band-path plane from its per-chunk owner lists (warp = row).
template <int DONLY>  // lr_fill_row's mode
__device__ __forceinline__ void band_fill_row(const RowArgs& ra, const BandArgs& a, FillSmem& sm, int64_t row,
                                              int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    const int W = a.W;
    const int p = (int)(row / a.H);
    const int64_t iR = row - (int64_t)p * a.H;
    const uint32_t gi = (uint32_t)(iR + 32 * a.band0);  // global row
    const int* bounds = a.cbound + ((int64_t)p * a.nb + iR / 32) * (kBandWarps + 1);
    int32_t* Drow = ra.D ? reinterpret_cast<int32_t*>(ra.D + p * ra.sD) + iR * W : nullptr;
    float* Srow = ra.S ? reinterpret_cast<float*>(ra.S + p * ra.sS) + iR * W : nullptr;
    int32_t* Lrow = ra.LB ? reinterpret_cast<int32_t*>(ra.LB + p * ra.sL) + iR * W : nullptr;
    int32_t* Nrow = ra.NC ? reinterpret_cast<int32_t*>(ra.NC + p * ra.sN) + iR * W : nullptr;
    // one round trip for the row's chunk bounds and list lengths, a second
    // one for all its lists (staged back to back when they fit together)
    const int bnd = lane <= kBandWarps ? __ldcg(bounds + lane) : 0;
    const int bnx = __shfl_down_sync(FULL, bnd, 1);
    const int ne = (lane < kBandWarps && bnd < bnx) ? __ldcg(a.nent + row * kBandWarps + lane) : 0;
    int off = ne;  // exclusive prefix over the chunks
#pragma unroll
    for (int o = 1; o < kBandWarps; o <<= 1) {
        const int v = __shfl_up_sync(FULL, off, o);
        if (lane >= o) off += v;
    }
    const int all = __shfl_sync(FULL, off, kBandWarps - 1);
    off -= ne;
    const bool staged = all <= kFillCap;
    __syncwarp();
    if (staged) {
#pragma unroll
        for (int w = 0; w < kBandWarps; ++w) {
            const int nE = __shfl_sync(FULL, ne, w), o = __shfl_sync(FULL, off, w);
            const int64_t at = row * a.Ws + __shfl_sync(FULL, bnd, w);
            for (int q = lane; q < nE; q += 32) {
                sm.e[o + q] = __ldcg(a.ent + at + q);
                sm.r[o + q] = __ldcg(a.entr + at + q);
            }
        }
        __syncwarp();
    }
    for (int w = 0; w < kBandWarps; ++w) {
        const int c0 = __shfl_sync(FULL, bnd, w), c1 = __shfl_sync(FULL, bnx, w);
        if (c0 >= c1) continue;
        const int nE = __shfl_sync(FULL, ne, w);
        const uint32_t* gE = a.ent + row * a.Ws + c0;
        const uint16_t* gR = a.entr + row * a.Ws + c0;
        if (staged) {
            const int o = __shfl_sync(FULL, off, w);
            lr_fill_row<DONLY>(ra, sm.e + o, sm.r + o, nE, gi, Drow, Srow, Lrow, Nrow, c0, c1, lane);
            continue;
        }
        if (nE <= kFillCap) {
            __syncwarp();
            for (int q = lane; q < nE; q += 32) {
                sm.e[q] = __ldcg(gE + q);
                sm.r[q] = __ldcg(gR + q);
            }
            __syncwarp();
            lr_fill_row<DONLY>(ra, sm.e, sm.r, nE, gi, Drow, Srow, Lrow, Nrow, c0, c1, lane);
            continue;
        }
        // a long list (dense stretches): 32-column blocks straight from L2
        int base = 0;
        for (int b = c0; b < c1; b += 32) {
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
            if (j < c1) {
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

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) with an mbarrier per buffer ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// generic-proxy accesses of shared memory before this point are ordered before
// later async-proxy (bulk copy) accesses of it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared, 16-byte aligned both sides, bytes a multiple of 16; completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Stacks and fill of one band in one CTA: the band's 8 warps build its rows'
// lists, then each writes 4 of its 32 rows.  The lists stay in L2; a CTA in
// its (latency-bound) stack phase shares the SM with CTAs in their (HBM-bound)
// fill phase (as two launches the phases took 156 + 766 us on C5, one launch gap more).  Fill phase per warp: the band's
// chunk bounds and the list lengths of its 4 rows in one round trip, then the
// rows' lists by TMA bulk copies into two buffers (row k + 2 is in flight while
// row k is written): no load latency between the rows' store streams.
struct FusedFill {
    uint32_t e[2][kFillCap];
    uint16_t r[2][kFillCap];
};

template <bool TAKE_NEW, int DONLY>
__global__ void __launch_bounds__(32 * kBandWarps, 4) k_band_rows_fill(RowArgs ra, BandArgs a) {
    extern __shared__ uint4 band_raw[];
    constexpr unsigned FULL = 0xffffffffu;
    const int64_t task = blockIdx.x;
    const int p = (int)(task / a.nb), b = (int)(task - (int64_t)p * a.nb);
    if (!band_plane(a, p)) return;  // CTA-uniform
    band_rows_body<TAKE_NEW>(a, *reinterpret_cast<BandSmem*>(band_raw), task);
    __syncthreads();  // the band's lists are written (global) and its shared memory is free
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    FusedFill& fs = reinterpret_cast<FusedFill*>(band_raw)[warp];
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<FusedFill*>(band_raw) + kBandWarps) + 2 * warp;
    const int nrows = min(32, a.H - 32 * b);
    const int nk = warp < nrows ? (nrows - warp + kBandWarps - 1) / kBandWarps : 0;  // this warp's rows (<= 4)
    static_assert(kBandWarps == 8, "lane = 8 * (row slot) + chunk");
    if (nk == 0) return;
    fence_proxy_async();  // this memory held the stack phase's lists (generic stores)
    if (lane == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
    }
    __syncwarp();
    const int64_t row0 = (int64_t)p * a.H + 32 * b + warp;  // rows row0 + 8 k
    const int* bounds = a.cbound + task * (kBandWarps + 1);
    const int bnd = lane <= kBandWarps ? __ldcg(bounds + lane) : 0;
    const int bnx = __shfl_down_sync(FULL, bnd, 1);
    // lane 8 k + w: row slot k, chunk w
    const int myk = lane >> 3, myw = lane & 7;
    const int wc0 = __shfl_sync(FULL, bnd, myw), wc1 = __shfl_sync(FULL, bnx, myw);
    const int ne = (myk < nk && wc0 < wc1) ? __ldcg(a.nent + (row0 + 8 * myk) * kBandWarps + myw) : 0;
    // staged offsets inside the row's buffer: multiples of 8 entries (16-byte aligned for both arrays)
    const int ne8 = (ne + 7) & ~7;
    int off = ne8;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const int v = __shfl_up_sync(FULL, off, o, 8);
        if (myw >= o) off += v;
    }
    const int tot = __shfl_sync(FULL, off, (lane & ~7) | 7);  // the row slot's total
    off -= ne8;
    if (__any_sync(FULL, tot > kFillCap)) {  // a row's lists do not fit a buffer: the synchronous path
        for (int k = 0; k < nk; ++k)
            band_fill_row<DONLY>(ra, a, *reinterpret_cast<FillSmem*>(&fs), row0 + 8 * k, lane);
        return;
    }
    auto issue = [&](int k, int buf) {  // row slot k's lists -> buffer buf
        const int t = __shfl_sync(FULL, tot, 8 * k);
        if (lane == 0) mbar_expect_tx(bars + buf, (uint32_t)t * 6u);
        __syncwarp();
        if (myk == k && ne > 0) {
            const int64_t at = (row0 + 8 * k) * a.Ws + wc0;
            bulk_g2s(fs.e[buf] + off, a.ent + at, (uint32_t)ne8 * 4u, bars + buf);
            bulk_g2s(fs.r[buf] + off, a.entr + at, (uint32_t)ne8 * 2u, bars + buf);
        }
    };
    issue(0, 0);
    if (nk > 1) issue(1, 1);
    int32_t* const Dp = ra.D ? reinterpret_cast<int32_t*>(ra.D + p * ra.sD) : nullptr;
    float* const Sp = ra.S ? reinterpret_cast<float*>(ra.S + p * ra.sS) : nullptr;
    int32_t* const Lp = ra.LB ? reinterpret_cast<int32_t*>(ra.LB + p * ra.sL) : nullptr;
    int32_t* const Np = ra.NC ? reinterpret_cast<int32_t*>(ra.NC + p * ra.sN) : nullptr;
    int waits[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (k >= nk) break;
        const int buf = k & 1;
        const int64_t row = row0 + 8 * k;
        {
            mbar_wait(bars + buf, (uint32_t)(waits[buf]++ & 1));  // the buffer's n-th armed use: phase parity n & 1
            const int64_t iR = row - (int64_t)p * a.H;
            const uint32_t gi = (uint32_t)(iR + 32 * a.band0);
            int32_t* Drow = Dp ? Dp + iR * a.W : nullptr;
            float* Srow = Sp ? Sp + iR * a.W : nullptr;
            int32_t* Lrow = Lp ? Lp + iR * a.W : nullptr;
            int32_t* Nrow = Np ? Np + iR * a.W : nullptr;
            for (int w = 0; w < kBandWarps; ++w) {
                const int c0 = __shfl_sync(FULL, bnd, w), c1 = __shfl_sync(FULL, bnx, w);
                if (c0 >= c1) continue;
                const int nE = __shfl_sync(FULL, ne, 8 * k + w), o = __shfl_sync(FULL, off, 8 * k + w);
                lr_fill_row<DONLY>(ra, fs.e[buf] + o, fs.r[buf] + o, nE, gi, Drow, Srow, Lrow, Nrow, c0, c1, lane);
            }
        }
        __syncwarp();  // the buffer's readers are done
        if (k + 2 < nk) issue(k + 2, buf);
    }
}

inline int band_fused_smem_bytes() {
    return std::max((int)sizeof(BandSmem), kBandWarps * ((int)sizeof(FusedFill) + 16));
}


}  // namespace dfc
