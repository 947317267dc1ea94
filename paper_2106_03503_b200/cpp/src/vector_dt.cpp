// vector_dt.cpp -- the drop-in's Danielsson transform over the C ABI
// (reference: vector_dt.cpp; the sweeps run in csrc/k_vector.cu).
#include "distfield/vector_dt.hpp"

#include <stdexcept>

#include "device.hpp"
#include "distfield/device_image.hpp"

namespace distfield {

std::string to_text(const OffsetMap& om) {
    std::string s;
    for (std::size_t i = 0; i < om.rows(); ++i) {
        for (std::size_t j = 0; j < om.cols(); ++j) {
            const Offset& o = om(i, j);
            if (j != 0) s.push_back(' ');
            if (o.is_set()) {
                s += std::to_string(o.dy);
                s.push_back(',');
                s += std::to_string(o.dx);
            } else {
                s += "inf";
            }
        }
        s.push_back('\n');
    }
    return s;
}

DistCache::DistCache(std::size_t side) : side_(side), memo_(side * side, -1) {
    if (side == 0) throw std::invalid_argument("cache side must be positive");
}

std::uint64_t DistCache::operator()(std::uint32_t a, std::uint32_t b) {
    if (a >= side_ || b >= side_) throw std::out_of_range("offset beyond cache extent");
    std::int64_t& v = memo_[static_cast<std::size_t>(a) * side_ + b];
    if (v < 0) {
        v = static_cast<std::int64_t>(a) * a + static_cast<std::int64_t>(b) * b;
        memo_[static_cast<std::size_t>(b) * side_ + a] = v;  // symmetric slot
    }
    return static_cast<std::uint64_t>(v);
}

namespace {

// d_img: rows x cols bytes in device memory, row pitch in bytes
VectorDtResult run_device(const std::uint8_t* d_img, std::size_t rows, std::size_t cols, std::size_t pitch,
                          bool first_only) {
    const std::size_t n = rows * cols;
    detail::DeviceBuffer<std::uint64_t> dd(n);
    detail::DeviceBuffer<std::uint32_t> dy(n), dx(n);
    detail::dfc_check(dfc_danielsson_u8(d_img, 1, (int64_t)rows, (int64_t)cols, (int64_t)pitch, 0, first_only ? 1 : 0,
                                        dd.get(), dy.get(), dx.get(), detail::stream()),
                      "danielsson");
    const std::vector<std::uint64_t> hd = dd.download();
    const std::vector<std::uint32_t> hy = dy.download(), hx = dx.download();
    VectorDtResult r{DistanceMap(rows, cols, DistanceKind::squared_euclidean), OffsetMap(rows, cols)};
    for (std::size_t i = 0; i < rows; ++i) {
        auto drow = r.distance.row(i);
        for (std::size_t j = 0; j < cols; ++j) {
            drow[j] = hd[i * cols + j];  // UINT64_MAX is DistanceMap::kInfinity
            r.offsets(i, j) = Offset{hy[i * cols + j], hx[i * cols + j]};
        }
    }
    return r;
}

VectorDtResult run(const BinaryImage& img, bool first_only) {
    auto dimg = detail::upload_image(img);
    return run_device(dimg.get(), img.rows(), img.cols(), img.pitch(), first_only);
}

}  // namespace

VectorDtResult danielsson(const BinaryImage& img) { return run(img, false); }
VectorDtResult danielsson_first_sweep(const BinaryImage& img) { return run(img, true); }
VectorDtResult danielsson(const DeviceImage& img) {
    return run_device(img.device_data(), img.rows(), img.cols(), img.cols(), false);
}

}  // namespace distfield
