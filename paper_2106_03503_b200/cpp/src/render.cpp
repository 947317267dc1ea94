// render.cpp -- to_gray / labels_to_gray (GPU, k_render.cu) and the
// plain-text dumps (host formatting) of the reference's grid.cpp:93-189,
// plus chamfer_normalized (propagation.cpp:111-127).
#include <cmath>
#include <cstdio>

#include "device.hpp"
#include "distfield/propagation.hpp"

namespace distfield {

using detail::DeviceBuffer;
using detail::dfc_check;
using detail::stream;

GrayImage to_gray(const DistanceMap& dm, GrayMapping mode) {
    const std::size_t n = dm.rows() * dm.cols();
    std::vector<std::int32_t> v(n);
    std::size_t p = 0;
    for (std::size_t i = 0; i < dm.rows(); ++i)
        for (std::uint64_t x : dm.row(i)) {
            if (!DistanceMap::is_infinite(x) && x > static_cast<std::uint64_t>(DFC_MAX_SQDIST))
                throw std::length_error("to_gray: value exceeds the device map range");
            v[p++] = DistanceMap::is_infinite(x) ? DFC_INF_I32 : static_cast<std::int32_t>(x);
        }
    DeviceBuffer<std::int32_t> d(n), mx(2);
    d.upload(v.data());
    DeviceBuffer<std::uint8_t> g(n);
    dfc_check(dfc_gray_i32(d.get(), (int64_t)n, mode == GrayMapping::sqrt_linear ? 1 : 0, g.get(), mx.get(),
                           reinterpret_cast<std::uint32_t*>(mx.get() + 1), stream()),
              "to_gray");
    const auto m = mx.download();
    if (m[0] < 0) throw std::domain_error("no features: distance map has no finite value");  // grid.cpp:95
    const auto h = g.download();
    GrayImage out(dm.rows(), dm.cols());
    std::copy(h.begin(), h.end(), out.cells().begin());
    return out;
}

GrayImage labels_to_gray(const LabelMap& labels, std::size_t feature_count) {
    if (feature_count == 0) throw std::domain_error("no features: empty label map");  // grid.cpp:113
    const std::size_t n = labels.rows() * labels.cols();
    std::vector<std::uint32_t> v(n);
    for (std::size_t i = 0, p = 0; i < labels.rows(); ++i)
        for (std::size_t j = 0; j < labels.cols(); ++j) v[p++] = labels(i, j);
    DeviceBuffer<std::uint32_t> d(n);
    d.upload(v.data());
    DeviceBuffer<std::uint8_t> g(n);
    dfc_check(dfc_labels_gray(d.get(), (int64_t)n, (int64_t)feature_count, g.get(), stream()), "labels_to_gray");
    const auto h = g.download();
    GrayImage out(labels.rows(), labels.cols());
    std::copy(h.begin(), h.end(), out.cells().begin());
    return out;
}

namespace {

template <typename Cell>
std::string matrix_text(std::size_t rows, std::size_t cols, Cell cell) {
    std::string out;
    for (std::size_t i = 0; i < rows; ++i) {
        for (std::size_t j = 0; j < cols; ++j) {
            if (j) out += ' ';
            cell(out, i, j);
        }
        out += '\n';
    }
    return out;
}

}  // namespace

std::string to_text(const DistanceMap& dm) {
    return matrix_text(dm.rows(), dm.cols(), [&](std::string& o, std::size_t i, std::size_t j) {
        const auto v = dm(i, j);
        o += DistanceMap::is_infinite(v) ? std::string("inf") : std::to_string(v);
    });
}

std::string to_text_sqrt(const DistanceMap& dm) {
    return matrix_text(dm.rows(), dm.cols(), [&](std::string& o, std::size_t i, std::size_t j) {
        const auto v = dm(i, j);
        if (DistanceMap::is_infinite(v)) {
            o += "inf";
            return;
        }
        char buf[48];
        std::snprintf(buf, sizeof buf, "%.6g", std::sqrt(static_cast<double>(v)));
        o += buf;
    });
}

std::string to_text(const Grid<double>& m) {
    return matrix_text(m.rows(), m.cols(), [&](std::string& o, std::size_t i, std::size_t j) {
        const double x = m(i, j);
        if (std::isinf(x)) {
            o += "inf";
            return;
        }
        const double r = std::round(x * 10.0) / 10.0;
        if (r == std::floor(r)) {
            o += std::to_string(static_cast<long long>(r));
        } else {
            char buf[48];
            std::snprintf(buf, sizeof buf, "%.1f", r);
            o += buf;
        }
    });
}

std::string to_text(const LabelMap& labels) {
    return matrix_text(labels.rows(), labels.cols(), [&](std::string& o, std::size_t i, std::size_t j) {
        const auto v = labels(i, j);
        o += v == LabelMap::kNoLabel ? std::string("inf") : std::to_string(v);
    });
}

Grid<double> chamfer_normalized(const DistanceMap& dm) {
    if (dm.kind() != DistanceKind::chamfer3) throw std::invalid_argument("chamfer_normalized requires a chamfer map");
    Grid<double> out(dm.rows(), dm.cols());
    for (std::size_t i = 0; i < dm.rows(); ++i)
        for (std::size_t j = 0; j < dm.cols(); ++j) {
            const auto v = dm(i, j);
            if (DistanceMap::is_infinite(v)) {
                out(i, j) = std::numeric_limits<double>::infinity();
            } else {
                const double d = static_cast<double>(v) / 3.0;
                out(i, j) = d * d;
            }
        }
    return out;
}

}  // namespace distfield
