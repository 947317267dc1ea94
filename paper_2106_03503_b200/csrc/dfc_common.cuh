// dfc_common.cuh -- shared device helpers for the distance-transform kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/distfield_cuda.h"

namespace dfc {

// "no object pixel in this column (band)" marker for uint16 row indices.
constexpr uint16_t kNoRow = 0xFFFF;
// Infinity inside the kernels (unsigned compare): every real value is < 2^31.
constexpr uint32_t kInfU = 0xFFFFFFFFu;
// Rows per band of the column pass: one bit per row in a 32-bit mask.
constexpr int kBand = 32;

// Per-thread error channel used by the C ABI.
struct Ctx {
    cudaStream_t stream;
    int launches = 0;
};

__device__ __forceinline__ uint32_t sq(uint32_t x) { return x * x; }

// Nearest object row to row i given the nearest row above (ra) and below
// (rb), kNoRow when absent.  Equal distances resolve to the UPPER row: the
// reference's fused vertical pass keeps the down-pass (upper) feature on a
// tie (exact_edt.cpp:327-360, strict '>' at :351).
__device__ __forceinline__ uint32_t pick_nearest(uint32_t i, uint32_t ra, uint32_t rb) {
    if (ra == kNoRow) return rb;
    if (rb == kNoRow) return ra;
    return (i - ra <= rb - i) ? ra : rb;
}

// floor(num / den) for 0 <= num < 2^32, 0 < den < 2^17, when the quotient is
// known to be < 2^16: approximate float quotient (MUFU.RCP) + one exact
// integer fix-up step each way (the estimate is off by at most one there).
// If the quotient would be >= 2^16 the result is only used after a range
// test has rejected it, so any value is fine.
__device__ __forceinline__ uint32_t small_udiv(uint32_t num, uint32_t den) {
    uint32_t q = __float2uint_rz(__fdividef(__uint2float_rn(num), __uint2float_rn(den)));
    int32_t r = (int32_t)(num - q * den);
    if (r < 0) { --q; r += (int32_t)den; }
    if (r >= (int32_t)den) ++q;
    return q;
}

// (float)sqrt((double)D) -- bit-identical to the reference's
// std::sqrt(static_cast<double>(v)) narrowed to float (grid.cpp:146).  For
// D < 2^24, (float)D is exact and RN(sqrt(D)) in float equals the double
// result narrowed (double rounding of sqrt is innocuous, 53 >= 2*24+2).
// Above, the float sqrt of the rounded D is within one ulp; it is fixed up
// with exact double arithmetic on the squared rounding midpoints (25-bit
// values, exact squares), which are never equal to an integer D.
__device__ __forceinline__ float dist_f32(uint32_t d) {
    if (d == (uint32_t)DFC_INF_I32 || d == kInfU) return __int_as_float(0x7f800000);
    float f = __fsqrt_rn(__uint2float_rn(d));
    if (d >= (1u << 24)) {
        const double dd = (double)d;
        const float up = __int_as_float(__float_as_int(f) + 1);
        const float dn = __int_as_float(__float_as_int(f) - 1);
        const double mu = 0.5 * ((double)f + (double)up), md = 0.5 * ((double)f + (double)dn);
        if (mu * mu < dd) f = up;
        else if (md * md > dd) f = dn;
    }
    return f;
}

}  // namespace dfc
