// propagation.cpp -- distfield raster transforms over the C ABI
// (reference: propagation.cpp:90-109; chessboard: tests/oracles.hpp:52-55).
#include "distfield/propagation.hpp"

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
    return detail::to_distance_map(d.download(), img.rows(), img.cols(), kind);
}

}  // namespace

DistanceMap cityblock_sequential(const BinaryImage& img) { return raster(img, DistanceKind::cityblock); }
DistanceMap cityblock_separable(const BinaryImage& img, unsigned) { return raster(img, DistanceKind::cityblock); }
DistanceMap chamfer34(const BinaryImage& img) { return raster(img, DistanceKind::chamfer3); }
DistanceMap chessboard(const BinaryImage& img) { return raster(img, DistanceKind::chessboard); }

}  // namespace distfield
