// k_rows_stream.cu -- stage 2 as a STREAMING scan: one lane = one row (chunk).
//
// Same result as k_rows.cu (the reference's envelope_rows / meijster_scan /
// voronoi label assembly, exact_edt.cpp:190-283, :362-369) with a different
// parallel decomposition: a warp owns 32 rows, every lane runs the reference's
// stack algorithm (exact_edt.cpp:208-223) over ITS row, left to right, in
// lockstep over columns -- all 32 lanes do the same work and no merges exist.
// Columns are final as soon as no later parabola can change their owner:
//
//     every parabola of a later column p >= m+1 has D_p(F) >= (m+1-F)^2, so
//     keep_old : D(F) <= (m+1-F)^2 => final   (a later column must be strictly smaller)
//     take_new : D(F) <  (m+1-F)^2 => final   (a later column wins ties)
//
// and stack entries owning only final columns leave the stack, so the live
// stack stays tiny in practice (<= ~50 entries on the five configs).  It lives
// in a per-lane ring in shared memory ([entry][lane]: each lane hits its own
// bank); a row that overflows its ring goes to a fallback list recomputed by
// k_rows.  tests/stream_model.py is the statement-level model (fuzzed against
// brute force for both tie rules).
//
// Chunks: a warp owns columns [c0, c1) of its 32 rows (blockIdx.y), so a row
// is scanned by W / chunk warps in parallel.  Each lane starts its scan at a
// warm-up column s0 <= c0 chosen so that no candidate left of s0 can own a
// column of the chunk (the bound is derived below), keeps the envelope over
// [F, W) with F starting at c0, and scans past c1 until its chunk is final.
//
// Data movement: nearest-row values are staged 32 rows x 32 columns at a time
// with coalesced 16-byte loads (prefetched one tile ahead).  A lane records the
// owner (column | nearest row << 16) of each final column in a 2 x 32-column
// staging slot; completed 32-column blocks are flushed by the whole warp --
// lane c computes column c of the block's row -- so D, sqrt(D), labels and
// nearest columns all leave with coalesced 128-byte stores.
#include "dfc_kernels.cuh"

namespace dfc {

constexpr int kSCap = 64;          // live-stack ring entries per lane
constexpr int kSEmit = 4;          // columns a lane may emit per scanned column (bounds the
                                   // lockstep cost of catch-up bursts; the backlog drains)
constexpr int kSTile = 32;         // columns per staged input tile
constexpr int kSTileStride = 34;   // halfwords per staged row (17 words: conflict-free)
constexpr int kSWarps = 2;         // warps (bands of 32 rows) per CTA
constexpr uint32_t kEmpty = 0xFFFF0000u;  // staged owner of a featureless row

enum : int { kOutD = 1, kOutS = 2, kOutL = 4, kOutN = 8 };

struct StreamSmem {
    uint16_t tile[32 * kSTileStride];   // input tile [row][col]
    uint2 stk[kSCap * 32];              // [entry][lane]: x = k | start << 16, y = nr_k
    uint32_t stage[2][32][33];          // [slot][lane][col]: owner k | nr_k << 16
};

template <bool TAKE_NEW, int OUTS>
__global__ void __launch_bounds__(32 * kSWarps) k_rows_stream(RowArgs a, int* fail_rows, int* fail_count,
                                                              int chunk) {
    extern __shared__ uint4 smem_raw[];
    StreamSmem& sm = reinterpret_cast<StreamSmem*>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int W = a.W;
    const int64_t band = (int64_t)blockIdx.x * kSWarps + (threadIdx.x >> 5);
    const int64_t row = band * 32 + lane;
    const bool active = row < a.total_rows;
    const int img = active ? (int)(row / a.H) : 0;
    const uint32_t i = active ? (uint32_t)(row - (int64_t)img * a.H) : 0u;
    const uint32_t gi = a.vdist ? 0u : i + (uint32_t)a.row0;
    const uint16_t* rowp = active ? a.nr + img * a.nr_img_stride + (int64_t)i * a.Wp : nullptr;
    // this warp's column chunk [c0, c1) (multiple of 32 wide)
    const int c0 = (int)blockIdx.y * chunk, c1 = min(c0 + chunk, W);

    // ---- staging: lane q loads 16-byte chunk (q & 3) of rows (q >> 2) + 8t ----
    uint4 pre[4];
    auto prefetch = [&](int c0) {
        const int j = c0 + 8 * (lane & 3);
        const int tt = j / a.tile_cols;  // column tile (all-to-all blocks); 8 | tile_cols
        const int64_t off = tt * a.tile_stride + (j - tt * a.tile_cols);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int rl = (lane >> 2) + 8 * t;
            const uint16_t* p = (const uint16_t*)__shfl_sync(0xffffffffu, (unsigned long long)rowp, rl);
            uint4 v = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
            if (p && j < W) v = __ldg(reinterpret_cast<const uint4*>(p + off));
            pre[t] = v;
        }
    };
    auto commit = [&]() {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int rl = (lane >> 2) + 8 * t;
            uint32_t* d = reinterpret_cast<uint32_t*>(sm.tile + rl * kSTileStride + 8 * (lane & 3));
            d[0] = pre[t].x; d[1] = pre[t].y; d[2] = pre[t].z; d[3] = pre[t].w;
        }
    };

    // ---- per-lane live stack + its two ends in registers ----
    int head = 0, cnt = 0;                  // ring entries head .. head+cnt-1
    int tk = 0, ts = 0; uint32_t tg = 0;    // top entry
    int bk = 0; uint32_t bnr = kNoRow, bg = 0; int bend = W;  // bottom entry, end of its range
    int F = c0;                             // first non-final column (columns < c0: other warps)
    uint32_t pend = 0;                      // staging slots holding a completed block
    bool dead = !active;                    // overflowed (or no row): recomputed elsewhere

    auto ent = [&](int idx) -> uint2& { return sm.stk[((head + idx) & (kSCap - 1)) * 32 + lane]; };
    auto load_bottom = [&]() {
        const uint2 e = ent(0);
        bk = (int)(e.x & 0xffffu);
        bnr = e.y;
        const uint32_t av = gi > bnr ? gi - bnr : bnr - gi;
        bg = av * av;
        bend = cnt >= 2 ? (int)(ent(1).x >> 16) : W;
    };

    // ---- warp-cooperative flush of completed 32-column blocks ----
    char* Dbase = a.D ? a.D + img * a.sD + (int64_t)i * W * 4 : nullptr;
    char* Sbase = a.S ? a.S + img * a.sS + (int64_t)i * W * 4 : nullptr;
    char* Lbase = a.LB ? a.LB + img * a.sL + (int64_t)i * W * 4 : nullptr;
    char* Nbase = a.NC ? a.NC + img * a.sN + (int64_t)i * W * 4 : nullptr;
    auto flush = [&](bool tail) {
        // tail: also write the partial block at the end of the row (F == W)
        uint32_t want = pend;
        if (tail && !dead && (c1 & 31) && F == c1) want |= 1u << ((c1 >> 5) & 1);
        uint32_t ready = __ballot_sync(0xffffffffu, want != 0);
        while (ready) {
            const int L = __ffs(ready) - 1;
            ready &= ready - 1;
            const uint32_t wL = __shfl_sync(0xffffffffu, want, L);
            const int FL = __shfl_sync(0xffffffffu, F, L);
            const uint32_t giL = __shfl_sync(0xffffffffu, gi, L);
            char* Db = (char*)__shfl_sync(0xffffffffu, (unsigned long long)Dbase, L);
            char* Sb = (char*)__shfl_sync(0xffffffffu, (unsigned long long)Sbase, L);
            char* Lb = (char*)__shfl_sync(0xffffffffu, (unsigned long long)Lbase, L);
            char* Nb = (char*)__shfl_sync(0xffffffffu, (unsigned long long)Nbase, L);
            for (int s = 0; s < 2; ++s) {
                if (!((wL >> s) & 1)) continue;
                // the block of parity s that ends at or before FL (or holds FL-1 at the tail)
                int b = (FL - 1) >> 5;
                if ((b & 1) != s) --b;
                const int j = 32 * b + lane;
                if (j >= W) continue;
                const uint32_t own = sm.stage[s][L][lane];
                const uint32_t k = own & 0xffffu, nr = own >> 16;
                const bool inf = nr == kNoRow;
                const uint32_t av = giL > nr ? giL - nr : nr - giL;
                const int dj = j - (int)k;
                const uint32_t d = inf ? (uint32_t)DFC_INF_I32 : av * av + (uint32_t)(dj * dj);
                if (OUTS & kOutD) __stcs(reinterpret_cast<int32_t*>(Db) + j, (int32_t)d);
                if (OUTS & kOutS) __stcs(reinterpret_cast<float*>(Sb) + j, dist_f32(d));
                if (OUTS & kOutL) __stcs(reinterpret_cast<int32_t*>(Lb) + j, inf ? -1 : (int32_t)(nr * (uint32_t)W + k));
                if (OUTS & kOutN) __stcs(reinterpret_cast<int32_t*>(Nb) + j, inf ? -1 : (int32_t)k);
            }
        }
        pend = 0;
    };

    // emit final columns F.. (bounded by m1 unless force); stops when the next
    // staging slot still holds an unflushed block
    auto finalize = [&](int m1, bool force) {
        for (;;) {
            bool blocked = false;
            int budget = force ? W : kSEmit;
            while (!dead && F < c1 && (force || F < m1) && budget-- > 0) {
                uint32_t own;
                if (cnt == 0) {
                    if (!force) break;  // no parabola yet: a later column will own these
                    own = kEmpty;       // end of a featureless row
                } else {
                    while (cnt >= 2 && bend <= F) {  // the bottom owns only final columns
                        head = (head + 1) & (kSCap - 1);
                        --cnt;
                        load_bottom();
                    }
                    if (!force) {
                        const uint32_t d = bg + (uint32_t)((F - bk) * (F - bk));
                        const uint32_t lim = (uint32_t)((m1 - F) * (m1 - F));
                        if (TAKE_NEW ? d >= lim : d > lim) break;
                    }
                    own = (uint32_t)bk | (bnr << 16);
                }
                const int s = (F >> 5) & 1;
                if ((pend >> s) & 1) { blocked = true; break; }
                sm.stage[s][lane][F & 31] = own;
                ++F;
                if ((F & 31) == 0) pend |= 1u << s;
            }
            if (__any_sync(0xffffffffu, pend != 0)) flush(false);
            if (!__any_sync(0xffffffffu, blocked)) break;
        }
    };

    // ---- warm-up start s0: no candidate left of s0 can own a column of the
    // chunk.  For a candidate F' >= c0 with vertical distance a', every F in
    // [c0, c1) has sqrt(D(F)) <= a' + |F - F'| <= A + (F - c0), A = min_F'
    // (a' + F' - c0); a column k <= s0 - 1 = c0 - A - 1 has (F - k)^2 >=
    // (A + F - c0 + 1)^2 > D(F).  So scanning from s0 = c0 - A is exact
    // (tests/stream_model.py::stream_chunk).  The pre-scan stops once F' - c0
    // reaches A; s0 = 0 when no candidate lies right of c0.
    int s0 = 0;
    if (c0 > 0) {
        int A = 0x3fffffff;
        bool need = !dead;
        for (int t0 = c0; t0 < W && __any_sync(0xffffffffu, need); t0 += kSTile) {
            prefetch(t0);
            __syncwarp();
            commit();
            __syncwarp();
            if (need) {
                for (int x = 0; x < kSTile && t0 + x < W && t0 + x - c0 < A; ++x) {
                    const uint32_t r = sm.tile[lane * kSTileStride + x];
                    if (r != kNoRow) {
                        const int am = (int)(gi > r ? gi - r : r - gi);
                        A = min(A, am + t0 + x - c0);
                    }
                }
                need = t0 + kSTile - c0 < A;
            }
            __syncwarp();
        }
        s0 = A >= 0x3fffffff ? 0 : max(0, c0 - A);
    }
    const int S0 = __reduce_min_sync(0xffffffffu, dead ? W : s0) & ~(kSTile - 1);

    if (S0 < W) prefetch(S0);
    for (int t0 = S0; t0 < W && __any_sync(0xffffffffu, !dead && F < c1); t0 += kSTile) {
        __syncwarp();
        commit();
        __syncwarp();
        if (t0 + kSTile < W) prefetch(t0 + kSTile);
        const int t1 = min(t0 + kSTile, W);
        for (int m = t0; m < t1; ++m) {
            const uint32_t r = sm.tile[lane * kSTileStride + (m - t0)];
            if (!dead && r != kNoRow && m >= s0) {
                const uint32_t am = gi > r ? gi - r : r - gi;
                const int gm = (int)(am * am);
                int start = -2;  // -2: stack empty -> owns from F
                while (cnt > 0) {
                    // num = v_m - v_k - k^2 + m^2 fits int32 (|.| < 2^31); ts*den < 2^32
                    const int num = gm - (int)tg + (m * m - tk * tk);
                    const uint32_t den = 2u * (uint32_t)(m - tk);
                    const uint32_t lim = (uint32_t)ts * den;
                    if (num < 0 || (TAKE_NEW ? (uint32_t)num <= lim : (uint32_t)num < lim)) {  // pop (:214)
                        if (--cnt > 0) {
                            const uint2 e = ent(cnt - 1);
                            tk = (int)(e.x & 0xffffu);
                            ts = (int)(e.x >> 16);
                            const uint32_t av = gi > e.y ? gi - e.y : e.y - gi;
                            tg = av * av;
                        }
                        continue;
                    }
                    const uint32_t lim2 = (uint32_t)(W - 1) * den;  // push iff start <= cols-1 (:218)
                    if (TAKE_NEW ? (uint32_t)num > lim2 : (uint32_t)num >= lim2) {
                        start = -1;
                    } else {
                        const uint32_t q = small_udiv((uint32_t)num, den);
                        start = TAKE_NEW ? (int)(q + ((uint32_t)num != q * den)) : (int)q + 1;
                    }
                    break;
                }
                if (start != -1) {
                    if (start < F) start = F;  // (also the empty-stack case, -2)
                    if (cnt == kSCap) {        // ring full: the fallback kernel redoes the row
                        dead = true;
                        fail_rows[atomicAdd(fail_count, 1)] = (int)row;
                    } else {
                        ent(cnt) = make_uint2((uint32_t)m | ((uint32_t)start << 16), r);
                        ++cnt;
                        tk = m;
                        ts = start;
                        tg = (uint32_t)gm;
                        if (cnt == 1) load_bottom();
                        else if (cnt == 2) bend = start;
                    }
                }
                if (cnt == 1) bend = W;
            }
            finalize(m + 1, false);
        }
    }
    finalize(W, true);  // no later columns: everything left is final
    flush(true);
}

template <bool TAKE_NEW>
inline const void* stream_kernel_ptr(int outs) {
    switch (outs) {
#define DFC_S(o) case o: return (const void*)k_rows_stream<TAKE_NEW, o>;
        DFC_S(1) DFC_S(2) DFC_S(3) DFC_S(4) DFC_S(5) DFC_S(6) DFC_S(7) DFC_S(8)
        DFC_S(9) DFC_S(10) DFC_S(11) DFC_S(12) DFC_S(13) DFC_S(14) DFC_S(15)
#undef DFC_S
        default: return nullptr;
    }
}

inline int stream_smem_bytes() { return kSWarps * (int)sizeof(StreamSmem); }

}  // namespace dfc
