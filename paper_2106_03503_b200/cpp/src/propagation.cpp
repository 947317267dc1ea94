// propagation.cpp -- distfield raster transforms over the C ABI
// (reference: propagation.cpp:90-109; chessboard: tests/oracles.hpp:52-55).
#include "distfield/propagation.hpp"

#include <algorithm>

#include "device.hpp"

namespace distfield {

namespace {

DistanceMap raster(const BinaryImage& img, DistanceKind kind) {
    auto dimg = detail::upload_image(img);
    detail::DeviceBuffer<std::int32_t> d(img.rows() * img.cols());
    int32_t* city = kind == DistanceKind::cityblock ? d.get() : nullptr;
    int32_t* chess = kind == DistanceKind::chessboard ? d.get() : nullptr;
    int32_t* cham = kind == DistanceKind::chamfer3 ? d.get() : nullptr;
    detail::dfc_check(dfc_raster_u8(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                                    city, chess, cham, detail::stream()),
                      "raster transform");
    return detail::to_distance_map(d, img.rows(), img.cols(), kind);
}

// one pass of dfc_raster_pass_u64 over the caller's map, in place
void pass(DistanceMap& dm, int which, const char* what) {
    const std::size_t rows = dm.rows(), cols = dm.cols();
    std::vector<std::uint64_t> host(rows * cols);
    for (std::size_t i = 0; i < rows; ++i) {
        const auto r = dm.row(i);
        std::copy(r.begin(), r.end(), host.begin() + static_cast<std::ptrdiff_t>(i * cols));
    }
    detail::DeviceBuffer<std::uint64_t> d(host.size());
    d.upload(host.data());
    detail::dfc_check(dfc_raster_pass_u64(d.get(), (int64_t)rows, (int64_t)cols, (int64_t)cols, which,
                                          detail::stream()),
                      what);
    host = d.download();
    for (std::size_t i = 0; i < rows; ++i) {
        auto r = dm.row(i);
        std::copy(host.begin() + static_cast<std::ptrdiff_t>(i * cols),
                  host.begin() + static_cast<std::ptrdiff_t>((i + 1) * cols), r.begin());
    }
}

}  // namespace

// propagation.cpp:16-58, 60-88
void cityblock_forward_pass(DistanceMap& dm) { pass(dm, DFC_PASS_CITYBLOCK_FORWARD, "cityblock_forward_pass"); }
void cityblock_backward_pass(DistanceMap& dm) { pass(dm, DFC_PASS_CITYBLOCK_BACKWARD, "cityblock_backward_pass"); }
void cityblock_vertical_passes(DistanceMap& dm, unsigned) {
    pass(dm, DFC_PASS_CITYBLOCK_VERTICAL, "cityblock_vertical_passes");
}
void cityblock_horizontal_passes(DistanceMap& dm, unsigned) {
    pass(dm, DFC_PASS_CITYBLOCK_HORIZONTAL, "cityblock_horizontal_passes");
}
void chamfer_forward_pass(DistanceMap& dm) { pass(dm, DFC_PASS_CHAMFER_FORWARD, "chamfer_forward_pass"); }
void chamfer_backward_pass(DistanceMap& dm) { pass(dm, DFC_PASS_CHAMFER_BACKWARD, "chamfer_backward_pass"); }

DistanceMap cityblock_sequential(const BinaryImage& img) { return raster(img, DistanceKind::cityblock); }
DistanceMap cityblock_separable(const BinaryImage& img, unsigned) { return raster(img, DistanceKind::cityblock); }
DistanceMap chamfer34(const BinaryImage& img) { return raster(img, DistanceKind::chamfer3); }
DistanceMap chessboard(const BinaryImage& img) { return raster(img, DistanceKind::chessboard); }

}  // namespace distfield
