// k_vector.cu -- Danielsson's vector transform (vector_dt.cpp:41-116): the
// approximate Euclidean transform that propagates offset MAGNITUDES (dy, dx)
// instead of distances, bit-exact with the reference's sequential sweeps.
//
// The reference is a strict raster recurrence: row i needs the FINISHED row
// i - 1 (sweep_down) or i + 1 (sweep_up), and inside a row the forward and the
// backward pass each carry a value from cell to cell.  What is parallel:
//
//  images  one CTA (4 warps) per image: batches run in parallel, a single image
//          is one CTA walking its rows.
//  pass V  the vertical update of a row (vector_dt.cpp:67-68): elementwise, all
//          warps; so are the row loads and stores.  Warp 0 carries passes F / B:
//  pass F/B  the carried value x reaches cell j as x + (0, j - s) from its
//          source cell s.  With base = the cell after pass V and c2 = the
//          diagonal neighbour's offset + (1, 1), the cell keeps the carried
//          value iff its squared length is below a threshold that does not
//          depend on x:
//              in-row neighbour applied first (:71-72, :88-89, :92-93):
//                  D1 < D(base) and D1 <= D(c2)
//              diagonal applied first (:75-76):  D1 < min(D(base), D(c2))
//          (strict updates, :58), and otherwise takes K = (D(c2) < D(base) ?
//          c2 : base), also independent of x, and becomes the new source.  So
//          a warp resolves 32 cells at a time: every lane tests the carried
//          value at its own cell, the first failing lane restarts the chain
//          with its K (a K equal to the carried value is no restart), and the
//          loop runs once per restart inside the block -- one step per 32
//          cells where one feature owns a stretch, one step per cell in the
//          worst case (the reference's own cost).
//
// The current and the previous row live in shared memory (or, for rows too
// wide for it, in a global scratch of the same layout); every finished row is
// written to the outputs, and the upward sweep reloads it from there.
#include "dfc_kernels.cuh"

namespace dfc {

constexpr uint64_t kDanInf = ~0ull;           // DistanceMap::kInfinity
constexpr uint32_t kDanUnset = 0xFFFFFFFFu;   // Offset::kUnset

struct DanArgs {
    const uint8_t* img;
    int64_t pitch, img_stride;   // bytes
    int rows, cols, Wb;          // Wb: row buffer stride (elements)
    int first_only;
    uint64_t* dist;              // [n][rows][cols]
    uint32_t* dy;
    uint32_t* dx;
    char* scratch;               // per image 2 row buffers (global), or null: shared memory
};

struct DanRow {
    uint64_t* D;
    uint32_t* y;
    uint32_t* x;
};

__device__ __forceinline__ uint64_t dan_sq(uint32_t a, uint32_t b) { return (uint64_t)a * a + (uint64_t)b * b; }

// One horizontal pass over 32 cells: lane = cell (valid lanes form a prefix).
// base / c2: the cell after the previous pass, and the diagonal candidate
// (kDanUnset in y: none); diag_first selects the threshold.  x*: the carried
// value at the cell before lane 0 (xs = its set flag).  Returns the cell's
// new state in (ry, rx, rD) and updates x* to the last valid lane's.
__device__ __forceinline__ void dan_block(bool valid, uint64_t Db, uint32_t by, uint32_t bx, uint64_t Dc, uint32_t cy,
                                          uint32_t cx, bool diag_first, bool& xs, uint32_t& xy, uint32_t& xx,
                                          uint64_t& rD, uint32_t& ry, uint32_t& rx, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    const bool take_c = Dc < Db;
    const uint64_t KD = take_c ? Dc : Db;
    const uint32_t Ky = take_c ? cy : by, Kx = take_c ? cx : bx;
    const bool Kset = Ky != kDanUnset;
    const uint64_t T = diag_first ? KD : (Db <= Dc ? Db : Dc + 1);  // min(Db, Dc) | min(Db, Dc + 1); Db > Dc: Dc finite
    rD = KD;
    ry = Ky;
    rx = Kx;
    const uint32_t vmask = __ballot_sync(FULL, valid);
    uint32_t rem = vmask;
    int src = -1;
    // self1: the cell would also restart if the cell before it had just restarted
    // (its K, moved one step, fails here too).  Cells on the far side of their
    // feature do that one after the other (the carried offset only grows), so a
    // whole run of them is taken in one step.
    uint32_t self1;
    {
        const uint32_t py = __shfl_up_sync(FULL, Ky, 1), px = __shfl_up_sync(FULL, Kx, 1);
        const uint32_t qx = px + 1u;
        const bool pset = py != kDanUnset;
        const bool ok = pset && (dan_sq(py, qx) < T || (Ky == py && Kx == qx));
        self1 = __ballot_sync(FULL, valid && lane > 0 && !ok);
    }
    while (rem) {
        if (!xs) {  // nothing carried: every cell keeps its K up to the first set one
            const uint32_t m = __ballot_sync(FULL, valid && Kset) & rem;
            if (m == 0) break;
            const int g = __ffs(m) - 1;
            xs = true;
            xy = __shfl_sync(FULL, Ky, g);
            xx = __shfl_sync(FULL, Kx, g);
            src = g;
            rem &= ~((2u << g) - 1u);
            continue;
        }
        const uint32_t cdx = xx + (uint32_t)(lane - src);
        const uint64_t D1 = dan_sq(xy, cdx);
        const bool in = (rem >> lane) & 1u;
        // a cell that keeps its own K breaks the chain only if K differs from the
        // carried value (inside one feature's region the vertical candidate and the
        // carried one are the same offset: the chain goes on unchanged)
        const bool same = Ky == xy && Kx == cdx;
        const uint32_t m = __ballot_sync(FULL, in && !(D1 < T) && !same) & rem;
        const int f = m ? __ffs(m) - 1 : 32;
        if (in && lane < f) {
            rD = D1;
            ry = xy;
            rx = cdx;
        }
        if (f == 32) break;
        // lane f restarts the chain with its K (possibly unset), and so do the
        // cells after it for which self1 holds without a gap: the chain goes on
        // from the last of them
        const uint32_t after = ~((2u << f) - 1u);           // lanes > f
        const uint32_t stop = ~self1 & after & vmask;        // first lane > f that does not restart by itself
        const int g = stop ? __ffs(stop) - 1 : 32;           // lanes f .. g - 1 keep their K
        const int s2 = min(g - 1, 31 - __clz(vmask));        // the new source (the last valid lane at most)
        xs = __shfl_sync(FULL, (int)Kset, s2) != 0;
        xy = __shfl_sync(FULL, Ky, s2);
        xx = __shfl_sync(FULL, Kx, s2);
        src = s2;
        rem &= ~((2u << s2) - 1u);
    }
    // the carried value for the next block: the last valid lane's result
    const int last = 31 - __clz(vmask);
    const uint32_t ly = __shfl_sync(FULL, ry, last), lx = __shfl_sync(FULL, rx, last);
    xs = ly != kDanUnset;
    xy = ly;
    xx = lx;
}

constexpr int kDanThreads = 128;  // warp 0 carries the row passes; all warps do the elementwise parts

__global__ void __launch_bounds__(kDanThreads) k_danielsson(DanArgs a) {
    extern __shared__ uint4 dan_raw[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int im = blockIdx.x;
    const int W = a.cols, H = a.rows, Wb = a.Wb;
    char* base = a.scratch ? a.scratch + (size_t)im * 2 * 16 * Wb : reinterpret_cast<char*>(dan_raw);
    DanRow buf[2];
    for (int b = 0; b < 2; ++b) {
        buf[b].D = reinterpret_cast<uint64_t*>(base) + (size_t)b * Wb;
        buf[b].y = reinterpret_cast<uint32_t*>(base + 16 * (size_t)Wb) + (size_t)b * Wb;
        buf[b].x = reinterpret_cast<uint32_t*>(base + 24 * (size_t)Wb) + (size_t)b * Wb;
    }
    const uint8_t* img = a.img + (size_t)im * a.img_stride;
    uint64_t* oD = a.dist + (size_t)im * H * W;
    uint32_t* oy = a.dy + (size_t)im * H * W;
    uint32_t* ox = a.dx + (size_t)im * H * W;

    auto init_row = [&](int i, DanRow r) {  // init_state, vector_dt.cpp:98-106
        const uint8_t* p = img + (size_t)i * a.pitch;
        for (int j = tid; j < W; j += kDanThreads) {
            const bool obj = p[j] != 0;
            r.D[j] = obj ? 0ull : kDanInf;
            r.y[j] = r.x[j] = obj ? 0u : kDanUnset;
        }
    };
    auto load_row = [&](int i, DanRow r) {
        for (int j = tid; j < W; j += kDanThreads) {
            r.D[j] = oD[(size_t)i * W + j];
            r.y[j] = oy[(size_t)i * W + j];
            r.x[j] = ox[(size_t)i * W + j];
        }
    };
    auto store_row = [&](int i, DanRow r) {
        for (int j = tid; j < W; j += kDanThreads) {
            oD[(size_t)i * W + j] = r.D[j];
            oy[(size_t)i * W + j] = r.y[j];
            ox[(size_t)i * W + j] = r.x[j];
        }
    };
    // one row of a sweep: cur from prev (the finished neighbouring row)
    auto row = [&](DanRow cur, DanRow prev, bool up) {
        for (int j = tid; j < W; j += kDanThreads) {  // vertical update (:67-68, :84-85)
            const uint32_t py = prev.y[j];
            if (py != kDanUnset) {
                const uint32_t ny = py + 1, nx = prev.x[j];
                const uint64_t d = dan_sq(ny, nx);
                if (cur.D[j] > d) {
                    cur.D[j] = d;
                    cur.y[j] = ny;
                    cur.x[j] = nx;
                }
            }
        }
        __syncthreads();
        if (W < 2 || tid >= 32) return;
        // forward (:69-73, :86-90): from the left neighbour, then from the diagonal one
        bool xs = cur.y[0] != kDanUnset;
        uint32_t xy = cur.y[0], xx = cur.x[0];
        for (int j0 = 1; j0 < W; j0 += 32) {
            const int j = j0 + lane;
            const bool valid = j < W;
            uint64_t Db = kDanInf, Dc = kDanInf;
            uint32_t by = kDanUnset, bx = kDanUnset, cy = kDanUnset, cx = kDanUnset;
            if (valid) {
                Db = cur.D[j];
                by = cur.y[j];
                bx = cur.x[j];
                const uint32_t py = prev.y[j - 1];
                if (py != kDanUnset) {
                    cy = py + 1;
                    cx = prev.x[j - 1] + 1;
                    Dc = dan_sq(cy, cx);
                }
            }
            uint64_t rD;
            uint32_t ry, rx;
            dan_block(valid, Db, by, bx, Dc, cy, cx, false, xs, xy, xx, rD, ry, rx, lane);
            if (valid) {
                cur.D[j] = rD;
                cur.y[j] = ry;
                cur.x[j] = rx;
            }
        }
        __syncwarp();
        // backward (:74-78 diagonal first; :91-95 in-row neighbour first)
        xs = cur.y[W - 1] != kDanUnset;
        xy = cur.y[W - 1];
        xx = cur.x[W - 1];
        for (int jh = W - 2; jh >= 0; jh -= 32) {
            const int j = jh - lane;
            const bool valid = j >= 0;
            uint64_t Db = kDanInf, Dc = kDanInf;
            uint32_t by = kDanUnset, bx = kDanUnset, cy = kDanUnset, cx = kDanUnset;
            if (valid) {
                Db = cur.D[j];
                by = cur.y[j];
                bx = cur.x[j];
                const uint32_t py = prev.y[j + 1];
                if (py != kDanUnset) {
                    cy = py + 1;
                    cx = prev.x[j + 1] + 1;
                    Dc = dan_sq(cy, cx);
                }
            }
            uint64_t rD;
            uint32_t ry, rx;
            dan_block(valid, Db, by, bx, Dc, cy, cx, !up, xs, xy, xx, rD, ry, rx, lane);
            if (valid) {
                cur.D[j] = rD;
                cur.y[j] = ry;
                cur.x[j] = rx;
            }
        }
        __syncwarp();
    };

    int c = 0;
    init_row(0, buf[c]);
    __syncthreads();
    store_row(0, buf[c]);
    for (int i = 1; i < H; ++i) {  // sweep_down (:64-79)
        init_row(i, buf[c ^ 1]);
        __syncthreads();
        row(buf[c ^ 1], buf[c], false);
        __syncthreads();
        store_row(i, buf[c ^ 1]);
        c ^= 1;
    }
    if (a.first_only) return;
    for (int i = H - 2; i >= 0; --i) {  // sweep_up (:81-96): buf[c] holds the finished row i + 1
        load_row(i, buf[c ^ 1]);
        __syncthreads();
        row(buf[c ^ 1], buf[c], true);
        __syncthreads();
        store_row(i, buf[c ^ 1]);
        c ^= 1;
    }
}

}  // namespace dfc
