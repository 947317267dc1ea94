// device_image.cpp -- GPU-resident images/maps for multi-step pipelines (the
// CLI path): packed P4 upload + device unpack, transforms into HBM, gray
// rendering on the device, downloads only on request.
#include "distfield/device_image.hpp"

#include "device.hpp"

namespace distfield {

using detail::cuda_check;
using detail::dfc_check;
using detail::stream;

namespace {

std::shared_ptr<void> device_alloc(std::size_t bytes) {
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, bytes + 16, stream()), "device alloc");
    return std::shared_ptr<void>(p, [](void* q) { cudaFreeAsync(q, stream()); });
}

template <typename T>
std::vector<T> download(const void* d, std::size_t n) {
    std::vector<T> h(n);
    cuda_check(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, stream()), "download");
    cuda_check(cudaStreamSynchronize(stream()), "synchronize");
    return h;
}

}  // namespace

DeviceImage::DeviceImage(std::size_t rows, std::size_t cols)
    : rows_(rows), cols_(cols), buf_(device_alloc(rows * cols)) {}

const std::uint8_t* DeviceImage::device_data() const { return static_cast<const std::uint8_t*>(buf_.get()); }

DeviceImage DeviceImage::from_raster(const PbmRaster& r, bool invert) {
    DeviceImage img(r.rows, r.cols);
    auto* dst = static_cast<std::uint8_t*>(img.buf_.get());
    if (r.packed) {  // 1/8 byte per pixel over the bus, unpacked in HBM
        detail::DeviceBuffer<std::uint8_t> bits(r.bytes.size());
        bits.upload(r.bytes.data());
        dfc_check(dfc_unpack_pbm(bits.get(), (int64_t)r.rows, (int64_t)r.cols, (int64_t)((r.cols + 7) / 8),
                                 invert ? 1 : 0, dst, (int64_t)r.cols, stream()),
                  "unpack P4 raster");
    } else {
        cuda_check(cudaMemcpyAsync(dst, r.bytes.data(), r.bytes.size(), cudaMemcpyHostToDevice, stream()), "upload");
        if (invert)
            dfc_check(dfc_binarize_u8(dst, (int64_t)r.rows, (int64_t)r.cols, (int64_t)r.cols, 1, dst,
                                      (int64_t)r.cols, stream()),
                      "invert");
    }
    return img;
}

DeviceImage DeviceImage::from_image(const BinaryImage& src, bool invert) {
    DeviceImage img(src.rows(), src.cols());
    auto* dst = static_cast<std::uint8_t*>(img.buf_.get());
    cuda_check(cudaMemcpyAsync(dst, src.data(), src.rows() * src.cols(), cudaMemcpyHostToDevice, stream()), "upload");
    if (invert)
        dfc_check(dfc_binarize_u8(dst, (int64_t)src.rows(), (int64_t)src.cols(), (int64_t)src.cols(), 1, dst,
                                  (int64_t)src.cols(), stream()),
                  "invert");
    return img;
}

std::size_t DeviceImage::object_count() const {
    auto cnt = device_alloc(sizeof(std::uint64_t));
    cuda_check(cudaMemsetAsync(cnt.get(), 0, sizeof(std::uint64_t), stream()), "memset");
    dfc_check(dfc_count_objects_u8(device_data(), (int64_t)rows_, (int64_t)cols_, (int64_t)cols_,
                                   static_cast<std::uint64_t*>(cnt.get()), stream()),
              "object_count");
    return static_cast<std::size_t>(download<std::uint64_t>(cnt.get(), 1)[0]);
}

DeviceMap::DeviceMap(std::size_t rows, std::size_t cols, DistanceKind kind)
    : rows_(rows), cols_(cols), kind_(kind), buf_(device_alloc(rows * cols * sizeof(std::int32_t))) {}

const std::int32_t* DeviceMap::device_data() const { return static_cast<const std::int32_t*>(buf_.get()); }

DistanceMap DeviceMap::download() const {
    return detail::to_distance_map(distfield::download<std::int32_t>(buf_.get(), rows_ * cols_), rows_, cols_, kind_);
}

GrayImage DeviceMap::to_gray(GrayMapping mode) const {
    const std::size_t n = rows_ * cols_;
    auto g = device_alloc(n);
    auto mx = device_alloc(2 * sizeof(std::int32_t));
    auto* mxp = static_cast<std::int32_t*>(mx.get());
    dfc_check(dfc_gray_i32(device_data(), (int64_t)n, mode == GrayMapping::sqrt_linear ? 1 : 0,
                           static_cast<std::uint8_t*>(g.get()), mxp, reinterpret_cast<std::uint32_t*>(mxp + 1),
                           stream()),
              "to_gray");
    if (distfield::download<std::int32_t>(mxp, 1)[0] < 0)
        throw std::domain_error("no features: distance map has no finite value");  // grid.cpp:95
    const auto h = distfield::download<std::uint8_t>(g.get(), n);
    GrayImage out(rows_, cols_);
    std::copy(h.begin(), h.end(), out.cells().begin());
    return out;
}

DeviceMap transform(const DeviceImage& img, DistanceKind kind) {
    DeviceMap m(img.rows(), img.cols(), kind);
    auto* d = static_cast<std::int32_t*>(m.buf_.get());
    const auto r = (int64_t)img.rows(), c = (int64_t)img.cols();
    if (kind == DistanceKind::squared_euclidean) {
        dfc_check(dfc_edt_u8(img.device_data(), r, c, c, DFC_BG_TO_OBJ, d, nullptr, nullptr, nullptr, stream()),
                  "edt");
    } else {
        dfc_check(dfc_raster_u8(img.device_data(), r, c, c, kind == DistanceKind::cityblock ? d : nullptr,
                                kind == DistanceKind::chessboard ? d : nullptr,
                                kind == DistanceKind::chamfer3 ? d : nullptr, stream()),
                  "raster transform");
    }
    return m;
}

DeviceLabels::DeviceLabels(std::size_t rows, std::size_t cols)
    : rows_(rows), cols_(cols), buf_(device_alloc(rows * cols * sizeof(std::uint32_t))) {}

LabelMap DeviceLabels::download() const {
    const auto h = distfield::download<std::uint32_t>(buf_.get(), rows_ * cols_);
    LabelMap lm(rows_, cols_);
    for (std::size_t i = 0; i < rows_; ++i)
        for (std::size_t j = 0; j < cols_; ++j) lm(i, j) = h[i * cols_ + j];
    return lm;
}

GrayImage DeviceLabels::to_gray(std::size_t feature_count) const {
    if (feature_count == 0) throw std::domain_error("no features: empty label map");  // grid.cpp:113
    const std::size_t n = rows_ * cols_;
    auto g = device_alloc(n);
    dfc_check(dfc_labels_gray(static_cast<const std::uint32_t*>(buf_.get()), (int64_t)n, (int64_t)feature_count,
                              static_cast<std::uint8_t*>(g.get()), stream()),
              "labels_to_gray");
    const auto h = distfield::download<std::uint8_t>(g.get(), n);
    GrayImage out(rows_, cols_);
    std::copy(h.begin(), h.end(), out.cells().begin());
    return out;
}

DeviceLabels voronoi_labels(const DeviceImage& img) {
    const std::size_t n = img.rows() * img.cols();
    const auto r = (int64_t)img.rows(), c = (int64_t)img.cols();
    DeviceLabels out(img.rows(), img.cols());
    auto dd = device_alloc(n * sizeof(std::int32_t));
    auto* lab = static_cast<std::int32_t*>(out.buf_.get());
    dfc_check(dfc_edt_u8(img.device_data(), r, c, c, DFC_BG_TO_OBJ, static_cast<std::int32_t*>(dd.get()), nullptr,
                         lab, nullptr, stream()),
              "voronoi_labels");
    if (download<std::int32_t>(dd.get(), 1)[0] == DFC_INF_I32)
        throw std::domain_error("no features: voronoi labels undefined");  // exact_edt.cpp:321
    dfc_check(dfc_label_ordinals(img.device_data(), r, c, c, lab, reinterpret_cast<std::uint32_t*>(lab), stream()),
              "voronoi_labels");
    return out;
}

}  // namespace distfield
