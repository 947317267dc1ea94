// k_passes.cu -- the reference's per-pass entry points over caller-owned
// uint64 / int64 maps, on the device:
//
//  k_row_owners  build_row_envelope / envelope_rows over ARBITRARY int64
//                vertical rows (exact_edt.cpp:190-283): per column j the owner
//                under the tie rule -- among column 0 (the envelope's base,
//                :208-210, kept even when it is a sentinel) and the columns
//                with vert < lmax (:212) -- and its value vert[k] + (j - k)^2.
//                The stack algorithm's integer boundaries (floor(x) + 1 for
//                keep_old, ceil(x) for take_new, :205) make the owner the
//                smallest (keep_old) or largest (take_new) minimiser, and the
//                minimisers are monotone in j (the parabolas are Monge), so
//                owners come from a divide and conquer over j: the owner of a
//                midpoint lies between its neighbours' owners; a warp scans
//                each midpoint's range (lane = candidate) and reduces.  O(W
//                log W) per row; every int64 value the reference accepts.
//  k_vpass_cb    cityblock_vertical_passes (propagation.cpp:36-46): per column,
//                the +1 relaxation down then up (thread = column, serial).
//  k_hpass_cb    cityblock_horizontal_passes (:48-58): per row, the +1
//                relaxation left to right then right to left = prefix / suffix
//                minima of d_k -/+ k (warp = row, shuffle scans).
//  k_raster_pass cityblock_forward/backward_pass (:16-34), chamfer_forward /
//                backward_pass (:60-88): a row depends on the finished previous
//                row, so ONE CTA walks the rows; within a row the relaxations
//                from the previous row are elementwise, and the chain along the
//                row (weight w) is a prefix minimum of t_k - w k (CTA scan).
//  relax(cell, nbr, w): an infinite neighbour never contributes, else cell =
//  min(cell, nbr + w) (propagation.cpp:10-12); maps hold values < 2^62.
#include "dfc_kernels.cuh"

namespace dfc {

constexpr uint64_t kInf64 = ~0ull;
constexpr int kOwnWarps = 8;

// (value, column) minimum over the warp with the tie rule on equal values
template <bool TAKE_NEW>
__device__ __forceinline__ void warp_best(int64_t& v, int& k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int k2 = __shfl_xor_sync(0xffffffffu, k, o);
        if (v2 < v || (v2 == v && (TAKE_NEW ? k2 > k : k2 < k))) {
            v = v2;
            k = k2;
        }
    }
}

template <bool TAKE_NEW>
__global__ void __launch_bounds__(32 * kOwnWarps) k_row_owners(const int64_t* __restrict__ vert, int64_t rows,
                                                             int cols, int64_t pitch, int64_t lmax,
                                                             int32_t* __restrict__ owner,
                                                             int64_t* __restrict__ value) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int64_t kNone = INT64_MAX;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t* v = vert + row * pitch;
        int32_t* own = owner + row * (int64_t)cols;
        // the best candidate for column j over [lo, hi] (candidates: 0 and vert < lmax)
        auto best = [&](int j, int lo, int hi, int64_t& bv, int& bk) {
            bv = kNone;
            bk = TAKE_NEW ? -1 : INT32_MAX;
            for (int k = lo + lane; k <= hi; k += 32) {
                const int64_t vk = __ldg(v + k);
                if (k != 0 && vk >= lmax) continue;
                const int64_t d = vk + (int64_t)(j - k) * (j - k);
                if (d < bv || (d == bv && (TAKE_NEW ? k > bk : k < bk))) {
                    bv = d;
                    bk = k;
                }
            }
            warp_best<TAKE_NEW>(bv, bk);
        };
        // the two ends, by full scans
        for (int e = warp; e < 2; e += kOwnWarps) {
            const int j = e == 0 ? 0 : cols - 1;
            int64_t bv;
            int bk;
            best(j, 0, cols - 1, bv, bk);
            if (lane == 0) {
                own[j] = bk;
                if (value) value[row * cols + j] = bv;
            }
        }
        __syncthreads();
        int P = 1;
        while (P < cols - 1) P <<= 1;
        // levels: midpoints j = s, 3s, 5s, ... (j < cols - 1) between computed neighbours
        for (int s = P >> 1; s >= 1; s >>= 1) {
            const int n = (cols - 1 - s + 2 * s - 1) / (2 * s);  // midpoints j = s (2t+1) < cols - 1
            for (int t = warp; t < n; t += kOwnWarps) {
                const int j = s * (2 * t + 1);
                const int lo = __ldcg(own + j - s);
                const int hi = __ldcg(own + min(j + s, cols - 1));
                int64_t bv;
                int bk;
                best(j, lo, hi, bv, bk);
                if (lane == 0) {
                    own[j] = bk;
                    if (value) value[row * cols + j] = bv;
                }
            }
            __syncthreads();
        }
    }
}

// cityblock_vertical_passes: thread = column
__global__ void k_vpass_cb(uint64_t* __restrict__ dm, int64_t rows, int64_t cols, int64_t pitch) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    uint64_t* c = dm + j;
    uint64_t prev = c[0];
    for (int64_t i = 1; i < rows; ++i) {
        uint64_t cur = c[i * pitch];
        if (prev != kInf64 && cur > prev + 1) {
            cur = prev + 1;
            c[i * pitch] = cur;
        }
        prev = cur;
    }
    prev = c[(rows - 1) * pitch];
    for (int64_t i = rows - 2; i >= 0; --i) {
        uint64_t cur = c[i * pitch];
        if (prev != kInf64 && cur > prev + 1) {
            cur = prev + 1;
            c[i * pitch] = cur;
        }
        prev = cur;
    }
}

// inclusive prefix minimum over the warp, lane order (inf = kInf64)
__device__ __forceinline__ int64_t warp_prefix_min(int64_t x, int lane, bool reverse) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = reverse ? __shfl_down_sync(0xffffffffu, x, o) : __shfl_up_sync(0xffffffffu, x, o);
        if (reverse ? lane + o < 32 : lane >= o) x = min(x, y);
    }
    return x;
}

// cityblock_horizontal_passes: warp = row.  Forward: d'_j = min_{k <= j,
// finite} d_k + (j - k) = j + prefix-min(d_k - k); backward likewise on d'.
__global__ void k_hpass_cb(uint64_t* __restrict__ dm, int64_t rows, int64_t cols, int64_t pitch) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += nw) {
        uint64_t* r = dm + i * pitch;
        constexpr int64_t kBig = INT64_MAX;
        for (int dir = 0; dir < 2; ++dir) {
            int64_t carry = kBig;  // running min of d_k -/+ k over the processed columns
            for (int64_t b = 0; b < cols; b += 32) {
                const int64_t j = dir == 0 ? b + lane : cols - 1 - (b + lane);
                const bool ok = b + lane < cols;
                const uint64_t d = ok ? r[j] : kInf64;
                const int64_t key = d == kInf64 ? kBig : (dir == 0 ? (int64_t)d - j : (int64_t)d + j);
                int64_t m = min(warp_prefix_min(key, lane, false), carry);
                carry = __shfl_sync(0xffffffffu, m, 31);
                if (ok && m != kBig) {
                    const uint64_t cand = (uint64_t)(dir == 0 ? m + j : m - j);
                    if (cand < d) r[j] = cand;
                }
            }
        }
    }
}

// One pass of the raster scans over the whole map; mode: 0 cityblock forward,
// 1 cityblock backward, 2 chamfer forward, 3 chamfer backward.  One CTA.
__global__ void __launch_bounds__(1024) k_raster_pass(uint64_t* __restrict__ dm, int64_t rows, int64_t cols,
                                                      int64_t pitch, int mode) {
    __shared__ int64_t wmin[32];
    const bool back = mode == 1 || mode == 3;
    const bool cham = mode >= 2;
    const int64_t wa = cham ? 3 : 1;          // axis weight (row chain and the previous row)
    const int64_t wd = 4;                     // diagonal weight (chamfer)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
    const int64_t per = (cols + nt - 1) / nt;  // columns per thread, in chain order
    constexpr int64_t kBig = INT64_MAX;
    for (int64_t s = 0; s < rows; ++s) {
        const int64_t i = back ? rows - 1 - s : s;
        uint64_t* r = dm + i * pitch;
        const uint64_t* p = s > 0 ? dm + (back ? i + 1 : i - 1) * pitch : nullptr;  // the finished row
        // t_j = min(d_j, p_j + wa, chamfer: p_{j-1} + 4, p_{j+1} + 4); then the chain
        // along the row (left to right forward, right to left backward):
        // d'_j = min over chain predecessors k of t_k + wa |j - k|
        int64_t local = kBig;  // the thread's running min of t_k - wa * pos_k (pos = chain index)
        const int64_t q0 = tid * per, q1 = min(cols, q0 + per);
        // pass 1: the chunk's minimum of t_k - wa * q
        for (int64_t q = q0; q < q1; ++q) {
            const int64_t j = back ? cols - 1 - q : q;
            uint64_t t = r[j];
            auto rel = [&](uint64_t nb, uint64_t w) {
                if (nb != kInf64 && t > nb + w) t = nb + w;
            };
            if (p) {
                rel(p[j], wa);
                if (cham) {
                    if (j > 0) rel(p[j - 1], wd);
                    if (j + 1 < cols) rel(p[j + 1], wd);
                }
            }
            if (t != kInf64) local = min(local, (int64_t)t - wa * q);
        }
        // exclusive prefix over the threads (chain order = thread order)
        int64_t inc = warp_prefix_min(local, lane, false);
        if (lane == 31) wmin[warp] = inc;
        int64_t exc = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) exc = kBig;
        __syncthreads();
        if (warp == 0) {
            const int nwarp = nt >> 5;
            int64_t w = lane < nwarp ? wmin[lane] : kBig;
            w = warp_prefix_min(w, lane, false);
            wmin[lane] = w;
        }
        __syncthreads();
        if (warp > 0) exc = min(exc, wmin[warp - 1]);
        // pass 2: apply, recomputing t (the previous row is untouched)
        int64_t run = exc;
        for (int64_t q = q0; q < q1; ++q) {
            const int64_t j = back ? cols - 1 - q : q;
            uint64_t t = r[j];
            auto rel = [&](uint64_t nb, uint64_t w) {
                if (nb != kInf64 && t > nb + w) t = nb + w;
            };
            if (p) {
                rel(p[j], wa);
                if (cham) {
                    if (j > 0) rel(p[j - 1], wd);
                    if (j + 1 < cols) rel(p[j + 1], wd);
                }
            }
            if (t != kInf64) run = min(run, (int64_t)t - wa * q);
            const uint64_t out = run == kBig ? kInf64 : (uint64_t)(run + wa * q);  // <= t
            if (out < r[j]) r[j] = out;
        }
        __syncthreads();  // row i is finished before row i +/- 1 reads it
    }
}

}  // namespace dfc
