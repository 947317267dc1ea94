// warmup.cpp -- the drop-in creates its CUDA context when the library is
// loaded, not inside the caller's first transform: context creation takes
// about a second on a cold GPU, and callers (the reference's own acceptance
// suite, proj/tests/acceptance.cpp:49-54) time their first call.
// DISTFIELD_NO_WARMUP=1 skips it.  Without a CUDA device this does nothing
// (the first transform then throws, as documented).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "distfield_cuda.h"

namespace {

struct Warmup {
    Warmup() {
        if (std::getenv("DISTFIELD_NO_WARMUP")) return;
        if (cudaFree(nullptr) != cudaSuccess) {  // creates the context
            cudaGetLastError();
            return;
        }
        // the stream-ordered pool and one kernel of libdfc (module load)
        std::int32_t* d = nullptr;
        if (cudaMallocAsync(reinterpret_cast<void**>(&d), 64, nullptr) == cudaSuccess) {
            cudaMemsetAsync(d, 0, 64, nullptr);
            dfc_sqrt_i32(d, reinterpret_cast<float*>(d + 8), 4, nullptr);
            cudaFreeAsync(d, nullptr);
            cudaStreamSynchronize(nullptr);
        }
        cudaGetLastError();
    }
};
const Warmup warmup;

}  // namespace
