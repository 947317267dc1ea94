// exact_edt.cpp -- distfield exact-EDT entry points over the C ABI.
// Reference behaviour followed: exact_edt.cpp:112-117 (vertical_pass),
// :232-237 (meijster_row_envelope), :272-283 (meijster_scan), :285-317 (edt),
// :319-371 (voronoi_labels).
#include "distfield/exact_edt.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "device.hpp"

namespace distfield {

using detail::DeviceBuffer;
using detail::dfc_check;
using detail::stream;

namespace {

// local_max (exact_edt.cpp:13-15): kind_bound + 1
std::int64_t local_max(std::size_t rows, std::size_t cols) {
    return static_cast<std::int64_t>(kind_bound(DistanceKind::squared_euclidean, rows, cols)) + 1;
}

// Vertical map -> uint16 vertical-distance plane (0xFFFF = no feature in the
// column); false when a finite value is not a perfect square (not a
// vertical-pass map: the generic path takes it).
bool vdist_plane(const DistanceMap& vert, std::size_t row0, std::size_t nrows, std::size_t pitch,
                 std::vector<std::uint16_t>& a) {
    a.assign(nrows * pitch, 0xFFFF);
    for (std::size_t i = 0; i < nrows; ++i) {
        const auto r = vert.row(row0 + i);
        for (std::size_t j = 0; j < vert.cols(); ++j) {
            const std::uint64_t v = r[j];
            if (DistanceMap::is_infinite(v)) continue;
            auto s = static_cast<std::uint64_t>(std::sqrt(static_cast<double>(v)));
            while (s * s > v) --s;
            while ((s + 1) * (s + 1) <= v) ++s;
            if (s * s != v || s >= 0xFFFF) return false;
            a[i * pitch + j] = static_cast<std::uint16_t>(s);
        }
    }
    return true;
}

// Per-column owners + values of int64 rows (load_row semantics done by the
// caller), tie rule as given: dfc_row_owners_i64.
void row_owners(const std::vector<std::int64_t>& rows_i64, std::size_t nrows, std::size_t cols, std::int64_t lmax,
                bool take_new, std::vector<std::int32_t>& owner, std::vector<std::int64_t>& value) {
    DeviceBuffer<std::int64_t> dv(rows_i64.size());
    dv.upload(rows_i64.data());
    DeviceBuffer<std::int32_t> dow(nrows * cols);
    DeviceBuffer<std::int64_t> dval(nrows * cols);
    dfc_check(dfc_row_owners_i64(dv.get(), (int64_t)nrows, (int64_t)cols, (int64_t)cols, lmax, take_new ? 1 : 0,
                                 dow.get(), dval.get(), stream()),
              "row envelope");
    owner = dow.download();
    value = dval.download();
}

struct Scan {
    std::vector<std::int32_t> d, col;  // d: DFC_INF_I32 = infinity; col: -1 = kNoColumn
};

Scan scan_rows(const DistanceMap& vert, std::size_t row0, std::size_t nrows) {
    const std::size_t cols = vert.cols(), pitch = cols + (cols & 1);
    std::vector<std::uint16_t> plane;
    if (vdist_plane(vert, row0, nrows, pitch, plane)) {
        DeviceBuffer<std::uint16_t> da(plane.size());
        da.upload(plane.data());
        DeviceBuffer<std::int32_t> dd(nrows * cols), dc(nrows * cols);
        dfc_check(dfc_envelope_vdist_u16(da.get(), (int64_t)nrows, (int64_t)cols, (int64_t)pitch, 1, dd.get(),
                                         nullptr, dc.get(), stream()),
                  "meijster_scan");
        return {dd.download(), dc.download()};
    }
    // any other map: load_row (exact_edt.cpp:29-35), the generic envelope,
    // store_value (:38-41) and the sentinel vertex rule (:278-279)
    const std::int64_t lmax = local_max(vert.rows(), cols);
    std::vector<std::int64_t> buf(nrows * cols);
    for (std::size_t i = 0; i < nrows; ++i) {
        const auto r = vert.row(row0 + i);
        for (std::size_t j = 0; j < cols; ++j)
            buf[i * cols + j] = DistanceMap::is_infinite(r[j]) ? lmax : static_cast<std::int64_t>(r[j]);
    }
    std::vector<std::int32_t> owner;
    std::vector<std::int64_t> value;
    row_owners(buf, nrows, cols, lmax, true, owner, value);
    Scan s{std::vector<std::int32_t>(nrows * cols), std::vector<std::int32_t>(nrows * cols)};
    for (std::size_t p = 0; p < nrows * cols; ++p) {
        const bool inf = value[p] >= lmax;
        s.d[p] = inf ? DFC_INF_I32 : static_cast<std::int32_t>(value[p]);
        s.col[p] = buf[(p / cols) * cols + static_cast<std::size_t>(owner[p])] >= lmax ? -1 : owner[p];
    }
    return s;
}

// (ks, js) of a row from its per-column owners (the runs of the owner row)
EnvelopeState envelope_from_owners(const std::int32_t* own, std::int64_t cols) {
    EnvelopeState env;
    env.ks.push_back(0);  // column-0 base (may own an empty segment)
    env.js.push_back(0);
    for (std::int64_t j = 0; j < cols; ++j) {
        const std::int32_t k = own[j];
        if (k < 0) break;  // featureless row: only the base, js = {0, cols}
        if (j == 0 && k == 0) continue;
        if (k != env.ks.back() || j == 0) {
            env.ks.push_back(k);
            env.js.push_back(j);
        }
    }
    env.js.push_back(cols);
    return env;
}

}  // namespace

namespace {
void vertical_direction(DistanceMap& dm, bool up) {
    const std::size_t rows = dm.rows(), cols = dm.cols();
    std::vector<std::uint64_t> host(rows * cols);
    for (std::size_t i = 0; i < rows; ++i) {
        const auto r = dm.row(i);
        std::copy(r.begin(), r.end(), host.begin() + static_cast<std::ptrdiff_t>(i * cols));
    }
    DeviceBuffer<std::uint64_t> d(host.size());
    d.upload(host.data());
    dfc_check(up ? dfc_vertical_up_pass_u64(d.get(), (int64_t)rows, (int64_t)cols, (int64_t)cols, stream())
                 : dfc_vertical_down_pass_u64(d.get(), (int64_t)rows, (int64_t)cols, (int64_t)cols, stream()),
              up ? "vertical_up_pass" : "vertical_down_pass");
    host = d.download();
    for (std::size_t i = 0; i < rows; ++i) {
        auto r = dm.row(i);
        std::copy(host.begin() + static_cast<std::ptrdiff_t>(i * cols),
                  host.begin() + static_cast<std::ptrdiff_t>((i + 1) * cols), r.begin());
    }
}
}  // namespace

// exact_edt.cpp:74-91
void vertical_down_pass(DistanceMap& dm, unsigned) { vertical_direction(dm, false); }

// exact_edt.cpp:93-110
void vertical_up_pass(DistanceMap& dm, unsigned) { vertical_direction(dm, true); }

DistanceMap vertical_pass(const BinaryImage& img, unsigned) {
    auto dimg = detail::upload_image(img);
    DeviceBuffer<std::int32_t> dv(img.rows() * img.cols());
    dfc_check(dfc_vertical_u8(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                              dv.get(), stream()),
              "vertical_pass");
    return detail::to_distance_map(dv, img.rows(), img.cols(), DistanceKind::squared_euclidean);
}

MeijsterResult meijster_scan(const DistanceMap& vert, ScanStats* stats, unsigned) {
    const Scan s = scan_rows(vert, 0, vert.rows());
    MeijsterResult out{detail::to_distance_map(s.d, vert.rows(), vert.cols(), DistanceKind::squared_euclidean),
                       Grid<std::uint32_t>(vert.rows(), vert.cols(), kNoColumn)};
    auto cells = out.nearest_col.cells();
    for (std::size_t p = 0; p < cells.size(); ++p)
        cells[p] = s.col[p] < 0 ? kNoColumn : static_cast<std::uint32_t>(s.col[p]);
    if (stats) stats->candidates += vert.rows() * vert.cols();
    return out;
}

// exact_edt.cpp:232-237: load_row + build_row_envelope(take_new)
EnvelopeState meijster_row_envelope(const DistanceMap& vert, std::size_t row) {
    if (row >= vert.rows()) throw std::out_of_range("meijster_row_envelope: row out of range");
    const std::int64_t lmax = local_max(vert.rows(), vert.cols());
    const auto r = vert.row(row);
    std::vector<std::int64_t> buf(r.size());
    for (std::size_t j = 0; j < r.size(); ++j)
        buf[j] = DistanceMap::is_infinite(r[j]) ? lmax : static_cast<std::int64_t>(r[j]);
    return build_row_envelope(buf, lmax, EnvelopeTie::take_new);
}

EnvelopeState build_row_envelope(std::span<const std::int64_t> vert, std::int64_t lmax, EnvelopeTie tie,
                                 ScanStats* stats) {
    const std::size_t cols = vert.size();
    if (cols == 0) {
        EnvelopeState env;
        env.ks.push_back(0);
        env.js = {0, 0};
        return env;
    }
    std::vector<std::int64_t> buf(vert.begin(), vert.end());
    std::vector<std::int32_t> owner;
    std::vector<std::int64_t> value;
    row_owners(buf, 1, cols, lmax, tie == EnvelopeTie::take_new, owner, value);
    if (stats) stats->candidates += cols;
    return envelope_from_owners(owner.data(), static_cast<std::int64_t>(cols));
}

DistanceMap edt(const BinaryImage& img, EdtAlgorithm, Orientation, ScanStats* stats, unsigned) {
    auto dimg = detail::upload_image(img);
    DeviceBuffer<std::int32_t> dd(img.rows() * img.cols());
    dfc_check(dfc_edt_u8(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                         DFC_BG_TO_OBJ, dd.get(), nullptr, nullptr, nullptr, stream()),
              "edt");
    if (stats) stats->candidates += img.rows() * img.cols();
    return detail::to_distance_map(dd, img.rows(), img.cols(), DistanceKind::squared_euclidean);
}

std::pair<DistanceMap, DistanceMap> edt_both_polarities(const BinaryImage& img) {
    auto dimg = detail::upload_image(img);
    const std::size_t n = img.rows() * img.cols();
    DeviceBuffer<std::int32_t> d0(n), d1(n);
    dfc_check(dfc_edt_u8_dual(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                              d0.get(), nullptr, d1.get(), nullptr, stream()),
              "edt_both_polarities");
    return {detail::to_distance_map(d0, img.rows(), img.cols(), DistanceKind::squared_euclidean),
            detail::to_distance_map(d1, img.rows(), img.cols(), DistanceKind::squared_euclidean)};
}

std::vector<float> edt_distances(const BinaryImage& img) {
    auto dimg = detail::upload_image(img);
    const std::size_t n = img.rows() * img.cols();
    DeviceBuffer<std::int32_t> dd(n);
    DeviceBuffer<float> ds(n);
    dfc_check(dfc_edt_u8(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                         DFC_BG_TO_OBJ, dd.get(), ds.get(), nullptr, nullptr, stream()),
              "edt_distances");
    return ds.download();
}

LabelMap voronoi_labels(const BinaryImage& img, unsigned) {
    const std::size_t n = img.rows() * img.cols();
    auto dimg = detail::upload_image(img);
    DeviceBuffer<std::int32_t> dd(n), dl(n);
    dfc_check(dfc_edt_u8(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                         DFC_BG_TO_OBJ, dd.get(), nullptr, dl.get(), nullptr, stream()),
              "voronoi_labels");
    std::int32_t d00 = 0;
    detail::cuda_check(cudaMemcpyAsync(&d00, dd.get(), sizeof d00, cudaMemcpyDeviceToHost, stream()), "d2h");
    detail::cuda_check(cudaStreamSynchronize(stream()), "synchronize");
    if (d00 == DFC_INF_I32) throw std::domain_error("no features: voronoi labels undefined");  // :321
    DeviceBuffer<std::uint32_t> dord(n);
    dfc_check(dfc_label_ordinals(dimg.get(), (int64_t)img.rows(), (int64_t)img.cols(), (int64_t)img.pitch(),
                                 dl.get(), dord.get(), stream()),
              "voronoi_labels");
    const auto ord = dord.download();
    LabelMap lm(img.rows(), img.cols());
    for (std::size_t i = 0; i < img.rows(); ++i)
        for (std::size_t j = 0; j < img.cols(); ++j) lm(i, j) = ord[i * img.cols() + j];
    return lm;
}

}  // namespace distfield
