// device.hpp -- plumbing between the value-semantics distfield API and the
// stream-ordered C ABI: a per-thread CUDA stream, RAII device buffers from the
// stream-ordered pool, status -> exception mapping, int32 -> uint64 maps.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
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

// Per-thread pinned bounce buffer: host <-> device copies of pageable caller
// memory (std::vector-backed grids) go through it at full PCIe rate and stay
// asynchronous; it only grows.
inline void* pinned(std::size_t bytes) {
    struct Pin {
        void* p = nullptr;
        std::size_t n = 0;
        ~Pin() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Pin pin;
    if (pin.n < bytes) {
        if (pin.p) cudaFreeHost(pin.p);
        pin.p = nullptr;
        pin.n = 0;
        if (cudaHostAlloc(&pin.p, bytes, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            pin.p = nullptr;
            return nullptr;  // the caller falls back to a pageable copy
        }
        pin.n = bytes;
    }
    return pin.p;
}

// f(begin, end) over [0, n) on the host threads (the reference's parallel_for,
// parallel.hpp:13-30, for the conversion loops of large maps).
template <typename F>
inline void host_parallel(std::size_t n, std::size_t grain, F f) {
    const std::size_t hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t nt = std::min<std::size_t>(hw, (n + grain - 1) / std::max<std::size_t>(grain, 1));
    if (nt <= 1) {
        f(std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    const std::size_t per = (n + nt - 1) / nt;
    for (std::size_t t = 0; t < nt; ++t) {
        const std::size_t b = t * per, e = std::min(n, b + per);
        if (b < e) th.emplace_back([=] { f(b, e); });
    }
    for (auto& x : th) x.join();
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
        const std::size_t bytes = n_ * sizeof(T);
        if (void* pin = pinned(bytes)) {  // staged: the bounce buffer is reused only after a synchronise
            std::memcpy(pin, host, bytes);
            cuda_check(cudaMemcpyAsync(p_, pin, bytes, cudaMemcpyHostToDevice, stream()), "upload");
            cuda_check(cudaStreamSynchronize(stream()), "synchronize");
            return;
        }
        cuda_check(cudaMemcpyAsync(p_, host, bytes, cudaMemcpyHostToDevice, stream()), "upload");
    }
    // The device values in the pinned bounce buffer (valid until this thread's
    // next upload / download), or nullptr when pinned memory is unavailable.
    const T* download_pinned() const {
        void* pin = pinned(n_ * sizeof(T));
        if (!pin) return nullptr;
        cuda_check(cudaMemcpyAsync(pin, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, stream()), "download");
        cuda_check(cudaStreamSynchronize(stream()), "synchronize");
        return static_cast<const T*>(pin);
    }
    std::vector<T> download() const {
        std::vector<T> h(n_);
        if (const T* pin = download_pinned()) {
            std::memcpy(h.data(), pin, n_ * sizeof(T));
            return h;
        }
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
inline DistanceMap to_distance_map(const std::int32_t* v, std::size_t rows, std::size_t cols, DistanceKind kind) {
    DistanceMap dm(rows, cols, kind);
    host_parallel(rows, std::max<std::size_t>(1, (std::size_t{1} << 18) / std::max<std::size_t>(cols, 1)),
                  [&](std::size_t r0, std::size_t r1) {
                      for (std::size_t i = r0; i < r1; ++i) {
                          auto r = dm.row(i);
                          const std::int32_t* src = v + i * cols;
                          for (std::size_t j = 0; j < cols; ++j)
                              r[j] = src[j] == DFC_INF_I32 ? DistanceMap::kInfinity : static_cast<std::uint64_t>(src[j]);
                      }
                  });
    return dm;
}
inline DistanceMap to_distance_map(const std::vector<std::int32_t>& v, std::size_t rows, std::size_t cols,
                                   DistanceKind kind) {
    return to_distance_map(v.data(), rows, cols, kind);
}
// Straight from the device: through the pinned bounce buffer when there is one.
inline DistanceMap to_distance_map(const DeviceBuffer<std::int32_t>& d, std::size_t rows, std::size_t cols,
                                   DistanceKind kind) {
    if (const std::int32_t* pin = d.download_pinned()) return to_distance_map(pin, rows, cols, kind);
    return to_distance_map(d.download(), rows, cols, kind);
}

}  // namespace distfield::detail
