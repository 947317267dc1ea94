// device.hpp -- plumbing between the value-semantics distfield API and the
// stream-ordered C ABI: a per-thread CUDA stream, RAII device buffers from the
// stream-ordered pool, status -> exception mapping, int32 -> uint64 maps.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "distfield/grid.hpp"
#include "distfield_cuda.h"

namespace distfield::detail {

inline cudaStream_t stream() {
    thread_local cudaStream_t s = [] {
        cudaStream_t st = nullptr;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
            throw std::runtime_error("distfield: no CUDA device available (the B200 path has no CPU fallback)");
        return st;
    }();
    return s;
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("distfield: ") + what + ": " + cudaGetErrorString(e));
}

inline void dfc_check(int status, const char* what) {
    if (status == DFC_OK) return;
    const std::string msg = std::string("distfield: ") + what + ": " + dfc_status_string(status);
    if (status == DFC_ERR_SHAPE) throw std::length_error(msg);
    if (status == DFC_ERR_ARG) throw std::invalid_argument(msg);
    if (status == DFC_ERR_NO_FEATURES) throw std::domain_error("no features: voronoi labels undefined");
    throw std::runtime_error(msg + " (cudaError " + std::to_string(dfc_last_cuda_error()) + ")");
}

template <typename T>
class DeviceBuffer {
public:
    explicit DeviceBuffer(std::size_t n) : n_(n) {
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T) + 16, stream()), "device alloc");
    }
    ~DeviceBuffer() {
        if (p_) cudaFreeAsync(p_, stream());
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
    T* get() const { return p_; }
    void upload(const T* host) {
        cuda_check(cudaMemcpyAsync(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice, stream()), "upload");
    }
    std::vector<T> download() const {
        std::vector<T> h(n_);
        cuda_check(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, stream()), "download");
        cuda_check(cudaStreamSynchronize(stream()), "synchronize");
        return h;
    }

private:
    T* p_ = nullptr;
    std::size_t n_;
};

inline DeviceBuffer<std::uint8_t> upload_image(const BinaryImage& img) {
    DeviceBuffer<std::uint8_t> d(img.rows() * img.cols());
    d.upload(img.data());
    return d;
}

// int32 GPU map (DFC_INF_I32 = infinity) -> reference DistanceMap (kInfinity).
inline DistanceMap to_distance_map(const std::vector<std::int32_t>& v, std::size_t rows, std::size_t cols,
                                   DistanceKind kind) {
    DistanceMap dm(rows, cols, kind);
    std::size_t p = 0;
    for (std::size_t i = 0; i < rows; ++i) {
        auto r = dm.row(i);
        for (std::size_t j = 0; j < cols; ++j, ++p)
            r[j] = v[p] == DFC_INF_I32 ? DistanceMap::kInfinity : static_cast<std::uint64_t>(v[p]);
    }
    return dm;
}

}  // namespace distfield::detail
