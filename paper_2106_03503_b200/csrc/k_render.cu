// k_render.cu -- the input/output epilogues of the CLI path, on the device so
// a bitmap goes host -> GPU as its packed raster and comes back only as the
// bytes the caller asked for.
//
//  * k_unpack_pbm   P4 raster (rows padded to whole bytes, MSB first, bit 1 =
//                   black = object; netpbm.cpp:81-95) -> uint8 0/1 image,
//                   optionally inverted (--polarity inside = img.inverted(),
//                   grid.cpp:38-44).  The upload shrinks 8x.
//  * k_binarize     uint8 image -> 0/1 (object = nonzero byte, grid.hpp:82),
//                   optionally inverted.
//  * k_count        object pixels (BinaryImage::object_count, grid.cpp:24-27).
//  * k_max_finite + k_gray   to_gray (grid.cpp:93-110): round(255 * v / max)
//                   or round(255 * sqrt(v) / sqrt(max)) in double, lround
//                   (half away from zero) exactly as the reference.
//  * k_labels_gray  labels_to_gray (grid.cpp:112-121): round(255 * id / n).
#include "dfc_kernels.cuh"

namespace dfc {

__global__ void k_unpack_pbm(const uint8_t* __restrict__ bits, int64_t rows, int64_t cols, int64_t row_bytes,
                             int invert, uint8_t* __restrict__ img, int64_t pitch) {
    const int64_t n = rows * row_bytes;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = p / row_bytes, b = p - i * row_bytes;
        const uint32_t byte = bits[p] ^ (invert ? 0xffu : 0u);
        uint8_t* dst = img + i * pitch + 8 * b;
        const int64_t nb = min((int64_t)8, cols - 8 * b);
        if (nb == 8 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
            uint32_t lo = 0, hi = 0;  // pixel 8b + t <- bit 7 - t
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                lo |= ((byte >> (7 - t)) & 1u) << (8 * t);
                hi |= ((byte >> (3 - t)) & 1u) << (8 * t);
            }
            *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
        } else {
            for (int t = 0; t < nb; ++t) dst[t] = (uint8_t)((byte >> (7 - t)) & 1u);
        }
    }
}

__global__ void k_binarize(const uint8_t* __restrict__ src, int64_t rows, int64_t cols, int64_t spitch, int invert,
                           uint8_t* __restrict__ dst, int64_t dpitch) {
    const int64_t n = rows * cols;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = p / cols, j = p - i * cols;
        dst[i * dpitch + j] = (uint8_t)((src[i * spitch + j] != 0) != (invert != 0));
    }
}

__global__ void k_count(const uint8_t* __restrict__ img, int64_t rows, int64_t cols, int64_t pitch,
                        unsigned long long* __restrict__ count) {
    const int64_t n = rows * cols;
    unsigned long long c = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = p / cols, j = p - i * cols;
        c += img[i * pitch + j] != 0;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// max finite value + 1 (0: no finite value) -- unsigned atomicMax friendly
__global__ void k_max_finite(const int32_t* __restrict__ d, int64_t n, unsigned int* __restrict__ mx1) {
    unsigned int m = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = d[p];
        if (v != DFC_INF_I32) m = max(m, (unsigned int)v + 1u);
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx1, m);
}

__global__ void k_gray(const int32_t* __restrict__ d, int64_t n, int sqrt_mode, const unsigned int* __restrict__ mx1,
                       uint8_t* __restrict__ out, int32_t* __restrict__ max_out) {
    const unsigned int m1 = *mx1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && max_out) *max_out = m1 == 0 ? -1 : (int32_t)(m1 - 1);
    const double mx = (double)(m1 == 0 ? 0u : m1 - 1u);
    const double denom = sqrt_mode ? sqrt(mx) : mx;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = d[p];
        uint8_t g = 0;
        if (m1 > 1) {  // max == 0 (or no finite value): all zeros (grid.cpp:97)
            if (v == DFC_INF_I32) {
                g = 255;   // unreachable for transform outputs (infinite only when all are)
            } else {
                const double x = sqrt_mode ? sqrt((double)v) : (double)v;
                g = (uint8_t)llround(255.0 * x / denom);
            }
        }
        out[p] = g;
    }
}

__global__ void k_labels_gray(const uint32_t* __restrict__ id, int64_t n, double count, uint8_t* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        out[p] = (uint8_t)llround(255.0 * (double)id[p] / count);
}

}  // namespace dfc
