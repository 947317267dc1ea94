// distfield/device_image.hpp -- B200 addition: images and maps that stay resident on
// the GPU between the steps of a pipeline (load -> transform -> render), the
// path the CLI (tools/distfield_b200.cpp) takes.  The value-semantics API
// (exact_edt.hpp, propagation.hpp) is built for one call per host image; this
// one uploads a P4 bitmap as its packed raster (1/8 byte per pixel), keeps
// the int32 maps in HBM and downloads only what is asked for.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>

#include "distfield/grid.hpp"
#include "distfield/vector_dt.hpp"
#include "distfield/netpbm.hpp"

namespace distfield {

// uint8 0/1 image in device memory (pitch == cols).
class DeviceImage {
public:
    // invert: BinaryImage::inverted() applied on the device (--polarity inside)
    static DeviceImage from_raster(const PbmRaster& raster, bool invert = false);
    static DeviceImage from_image(const BinaryImage& img, bool invert = false);

    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    const std::uint8_t* device_data() const;
    std::size_t object_count() const;  // counted on the GPU (synchronises)

private:
    DeviceImage(std::size_t rows, std::size_t cols);
    std::size_t rows_, cols_;
    std::shared_ptr<void> buf_;
};

// int32 distance map in device memory (DFC_INF_I32 = infinity).
class DeviceMap {
public:
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    DistanceKind kind() const { return kind_; }
    const std::int32_t* device_data() const;

    DistanceMap download() const;
    GrayImage to_gray(GrayMapping mode) const;  // std::domain_error if no finite value

private:
    friend DeviceMap transform(const DeviceImage&, DistanceKind);
    DeviceMap(std::size_t rows, std::size_t cols, DistanceKind kind);
    std::size_t rows_, cols_;
    DistanceKind kind_;
    std::shared_ptr<void> buf_;
};

// squared_euclidean (edt), cityblock, chessboard or chamfer3 of the image.
DeviceMap transform(const DeviceImage& img, DistanceKind kind);

// Danielsson's vector transform of an image already in device memory
// (vector_dt.hpp; the CLI's --algorithm danielsson): host result.
VectorDtResult danielsson(const DeviceImage& img);

// Voronoi labels (ordinals, the reference LabelMap) on the device; throws
// std::domain_error("no features: voronoi labels undefined") for an image
// without objects (exact_edt.cpp:321).
class DeviceLabels {
public:
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    LabelMap download() const;
    GrayImage to_gray(std::size_t feature_count) const;

private:
    friend DeviceLabels voronoi_labels(const DeviceImage&);
    DeviceLabels(std::size_t rows, std::size_t cols);
    std::size_t rows_, cols_;
    std::shared_ptr<void> buf_;
};

DeviceLabels voronoi_labels(const DeviceImage& img);

}  // namespace distfield
