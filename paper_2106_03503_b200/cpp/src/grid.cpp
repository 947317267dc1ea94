// grid.cpp -- host-side helpers of the drop-in core types (not on the GPU
// path: construction, enumeration and small utilities, grid.hpp).
#include "distfield/grid.hpp"

#include <algorithm>
#include <string>

namespace distfield {

BinaryImage BinaryImage::from_points(std::size_t rows, std::size_t cols, std::span<const GridPoint> points) {
    BinaryImage img(rows, cols);
    for (const GridPoint& p : points) {
        if (p.row >= rows || p.col >= cols)
            throw std::out_of_range("point (" + std::to_string(p.row) + ", " + std::to_string(p.col) +
                                    ") outside " + std::to_string(rows) + "x" + std::to_string(cols) + " image");
        img.set_object(p.row, p.col);
    }
    return img;
}

std::size_t BinaryImage::object_count() const {
    return static_cast<std::size_t>(std::count_if(px_.cells().begin(), px_.cells().end(),
                                                  [](std::uint8_t c) { return c != 0; }));
}

std::vector<FeaturePoint> BinaryImage::feature_points() const {
    std::vector<FeaturePoint> pts;
    std::uint32_t ordinal = 0;
    const auto cells = px_.cells();
    for (std::size_t p = 0; p < cells.size(); ++p)
        if (cells[p]) pts.push_back({p / cols(), p % cols(), ordinal++});
    return pts;
}

BinaryImage BinaryImage::inverted() const {
    BinaryImage out(rows(), cols());
    auto dst = out.px_.cells();
    const auto src = px_.cells();
    for (std::size_t p = 0; p < src.size(); ++p) dst[p] = src[p] ? 0 : 1;
    return out;
}

BinaryImage BinaryImage::transposed() const {
    BinaryImage out(cols(), rows());
    out.px_ = px_.transposed();
    return out;
}

std::uint64_t kind_bound(DistanceKind kind, std::size_t rows, std::size_t cols) {
    const std::uint64_t h = rows - 1, w = cols - 1;
    switch (kind) {
        case DistanceKind::cityblock: return h + w;
        case DistanceKind::chessboard: return std::max(h, w);
        case DistanceKind::chamfer3: return 4 * (h + w);
        case DistanceKind::squared_euclidean: return h * h + w * w;
    }
    throw std::invalid_argument("unknown distance kind");
}

bool DistanceMap::all_infinite() const {
    return std::all_of(v_.cells().begin(), v_.cells().end(), is_infinite);
}

std::optional<std::uint64_t> DistanceMap::max_finite() const {
    std::optional<std::uint64_t> m;
    for (std::uint64_t v : v_.cells())
        if (!is_infinite(v)) m = m ? std::max(*m, v) : v;
    return m;
}

DistanceMap DistanceMap::transposed() const {
    DistanceMap out(cols(), rows(), kind_);
    out.v_ = v_.transposed();
    return out;
}

DistanceMap init_distance_map(const BinaryImage& img, DistanceKind kind) {
    DistanceMap dm(img.rows(), img.cols(), kind);
    const std::uint8_t* px = img.data();
    for (std::size_t i = 0; i < img.rows(); ++i) {
        auto r = dm.row(i);
        for (std::size_t j = 0; j < img.cols(); ++j)
            if (px[i * img.cols() + j]) r[j] = 0;
    }
    return dm;
}

}  // namespace distfield
