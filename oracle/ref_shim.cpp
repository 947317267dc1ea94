// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat extern "C" shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile directly from the reference sources where they lie
// (/root/reference/proj/core/src/{grid,exact_edt,propagation,random_image,netpbm,vector_dt}.cpp)
// into oracle/_ref/libdfref.so.  Used (a) to pin the C restatement
// oracle/dt_oracle.c and (b) as bench.py's CPU baseline ("kind": "reference").
// Each call copies the caller's uint8 buffer into a distfield::BinaryImage
// outside the timed region and reports the wall time of the reference call
// alone (steady_clock) through *ns.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <span>
#include <string>

#include "distfield/exact_edt.hpp"
#include "distfield/grid.hpp"
#include "distfield/netpbm.hpp"
#include "distfield/propagation.hpp"
#include "distfield/random_image.hpp"
#include "distfield/vector_dt.hpp"

using namespace distfield;

namespace {

BinaryImage to_image(const std::uint8_t* img, std::size_t rows, std::size_t cols) {
    BinaryImage out(rows, cols);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j)
            if (img[i * cols + j]) out.set_object(i, j);
    return out;
}

void copy_map(const DistanceMap& dm, std::uint64_t* out) {
    const auto cells = dm.values().cells();
    std::memcpy(out, cells.data(), cells.size() * sizeof(std::uint64_t));
}

using clk = std::chrono::steady_clock;
double since(clk::time_point t0) {
    return std::chrono::duration<double, std::nano>(clk::now() - t0).count();
}

}  // namespace

extern "C" {

int dfref_generate_random_image(std::size_t rows, std::size_t cols, double density,
                                std::uint64_t seed, std::uint8_t* out) {
    const auto img = generate_random_image(rows, cols, density, seed);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) out[i * cols + j] = img.is_object(i, j) ? 1 : 0;
    return 0;
}

// edt(img, algorithm, orientation, stats, threads); algorithm 0..3 =
// bruteforce/simple/improved/envelope, orient 0..2 = automatic/rows/columns.
int dfref_edt(const std::uint8_t* img, std::size_t rows, std::size_t cols, int algorithm,
              int orient, unsigned threads, std::uint64_t* out, std::uint64_t* candidates,
              double* ns) {
    const auto bi = to_image(img, rows, cols);
    ScanStats stats;
    const auto t0 = clk::now();
    const auto dm = edt(bi, static_cast<EdtAlgorithm>(algorithm), static_cast<Orientation>(orient),
                        candidates ? &stats : nullptr, threads);
    if (ns) *ns = since(t0);
    if (out) copy_map(dm, out);
    if (candidates) *candidates = stats.candidates;
    return 0;
}

int dfref_vertical_pass(const std::uint8_t* img, std::size_t rows, std::size_t cols,
                        std::uint64_t* out) {
    copy_map(vertical_pass(to_image(img, rows, cols)), out);
    return 0;
}

int dfref_meijster_scan(const std::uint8_t* img, std::size_t rows, std::size_t cols,
                        std::uint64_t* out, std::uint32_t* nearest_col) {
    const auto res = meijster_scan(vertical_pass(to_image(img, rows, cols)));
    copy_map(res.map, out);
    const auto nc = res.nearest_col.cells();
    std::memcpy(nearest_col, nc.data(), nc.size() * sizeof(std::uint32_t));
    return 0;
}

// meijster_row_envelope(vertical_pass(img), row); returns ks.size() (js has one more).
long long dfref_row_envelope(const std::uint8_t* img, std::size_t rows, std::size_t cols,
                             std::size_t row, std::int64_t* ks, std::int64_t* js) {
    const auto env = meijster_row_envelope(vertical_pass(to_image(img, rows, cols)), row);
    for (std::size_t t = 0; t < env.ks.size(); ++t) ks[t] = env.ks[t];
    for (std::size_t t = 0; t < env.js.size(); ++t) js[t] = env.js[t];
    return static_cast<long long>(env.ks.size());
}

// build_row_envelope on an arbitrary int64 row (exact_edt.hpp:71-72).
long long dfref_build_row_envelope(const std::int64_t* vert, std::size_t cols, std::int64_t lmax, int take_new,
                                   std::int64_t* ks, std::int64_t* js) {
    const auto env = build_row_envelope(std::span<const std::int64_t>(vert, cols), lmax,
                                        take_new ? EnvelopeTie::take_new : EnvelopeTie::keep_old);
    for (std::size_t t = 0; t < env.ks.size(); ++t) ks[t] = env.ks[t];
    for (std::size_t t = 0; t < env.js.size(); ++t) js[t] = env.js[t];
    return static_cast<long long>(env.ks.size());
}

// One per-pass in-place function (propagation.hpp:15-26) over a uint64 map.
void dfref_raster_pass(std::uint64_t* map, std::size_t rows, std::size_t cols, int pass) {
    DistanceMap dm(rows, cols, DistanceKind::cityblock);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) dm(i, j) = map[i * cols + j];
    switch (pass) {
        case 0: cityblock_forward_pass(dm); break;
        case 1: cityblock_backward_pass(dm); break;
        case 2: cityblock_vertical_passes(dm, 1); break;
        case 3: cityblock_horizontal_passes(dm, 1); break;
        case 4: chamfer_forward_pass(dm); break;
        default: chamfer_backward_pass(dm); break;
    }
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) map[i * cols + j] = dm(i, j);
}

// voronoi_labels; returns -1 where the reference throws std::domain_error.
int dfref_voronoi_labels(const std::uint8_t* img, std::size_t rows, std::size_t cols,
                         unsigned threads, std::uint32_t* labels, double* ns) {
    const auto bi = to_image(img, rows, cols);
    try {
        const auto t0 = clk::now();
        const auto lm = voronoi_labels(bi, threads);
        if (ns) *ns = since(t0);
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t j = 0; j < cols; ++j) labels[i * cols + j] = lm(i, j);
    } catch (const std::domain_error&) {
        return -1;
    }
    return 0;
}

// edt + voronoi_labels over a batch of n same-shape images (C3 baseline).
int dfref_edt_labels_batch(const std::uint8_t* imgs, std::size_t n, std::size_t rows,
                           std::size_t cols, unsigned threads, std::uint64_t* dist,
                           std::uint32_t* labels, double* ns) {
    double total = 0.0;
    int status = 0;
    for (std::size_t b = 0; b < n; ++b) {
        const auto bi = to_image(imgs + b * rows * cols, rows, cols);
        const auto t0 = clk::now();
        const auto dm = edt(bi, EdtAlgorithm::envelope, Orientation::automatic, nullptr, threads);
        try {
            const auto lm = voronoi_labels(bi, threads);
            total += since(t0);
            if (labels)
                for (std::size_t i = 0; i < rows; ++i)
                    for (std::size_t j = 0; j < cols; ++j)
                        labels[b * rows * cols + i * cols + j] = lm(i, j);
        } catch (const std::domain_error&) {
            total += since(t0);
            status = -1;
        }
        if (dist) copy_map(dm, dist + b * rows * cols);
    }
    if (ns) *ns = total;
    return status;
}

// kind: 0 cityblock_sequential, 1 cityblock_separable(threads), 2 chamfer34.
int dfref_propagation(const std::uint8_t* img, std::size_t rows, std::size_t cols, int kind,
                      unsigned threads, std::uint64_t* out, double* ns) {
    const auto bi = to_image(img, rows, cols);
    const auto t0 = clk::now();
    DistanceMap dm = kind == 0   ? cityblock_sequential(bi)
                     : kind == 1 ? cityblock_separable(bi, threads)
                                 : chamfer34(bi);
    if (ns) *ns = since(t0);
    copy_map(dm, out);
    return 0;
}

// ---- the CLI's I/O layer (checkers for tools/distfield_b200) ----

static int put_text(const std::string& t, char* out, std::size_t cap) {
    if (out && cap > t.size()) std::memcpy(out, t.c_str(), t.size() + 1);
    return static_cast<int>(t.size());
}

// read_netpbm: 0 and the image (out may be NULL to query rows/cols), or 1 and
// the NetpbmError message (with its byte offset) in err.
int dfref_read_netpbm(const char* bytes, std::size_t n, std::uint8_t* out, std::size_t* rows, std::size_t* cols,
                      char* err, std::size_t errcap) {
    try {
        const auto img = read_netpbm(std::string_view(bytes, n));
        *rows = img.rows();
        *cols = img.cols();
        if (out)
            for (std::size_t i = 0; i < img.rows(); ++i)
                for (std::size_t j = 0; j < img.cols(); ++j) out[i * img.cols() + j] = img.is_object(i, j);
        return 0;
    } catch (const std::exception& e) {
        put_text(e.what(), err, errcap);
        return 1;
    }
}

// write_netpbm(BinaryImage, variant 0 plain / 1 raw) -> bytes; returns size.
int dfref_write_pbm(const std::uint8_t* img, std::size_t rows, std::size_t cols, int raw, char* out,
                    std::size_t cap) {
    const std::string t = write_netpbm(to_image(img, rows, cols), raw ? PbmVariant::raw : PbmVariant::plain);
    if (out && cap >= t.size()) std::memcpy(out, t.data(), t.size());
    return static_cast<int>(t.size());
}

static DistanceMap ref_transform(const BinaryImage& bi, int metric) {
    return metric == 0   ? edt(bi, EdtAlgorithm::envelope)
           : metric == 1 ? cityblock_sequential(bi)
                         : chamfer34(bi);
}

// Text dump of a transform: metric 0 edt / 1 cityblock / 2 chamfer34;
// mode 0 to_text, 1 to_text_sqrt, 2 to_text(chamfer_normalized).  Returns
// the length (the text is written when cap > length).
int dfref_transform_text(const std::uint8_t* img, std::size_t rows, std::size_t cols, int metric, int mode,
                         char* out, std::size_t cap) {
    const DistanceMap dm = ref_transform(to_image(img, rows, cols), metric);
    return put_text(mode == 0 ? to_text(dm) : mode == 1 ? to_text_sqrt(dm) : to_text(chamfer_normalized(dm)), out,
                    cap);
}

// to_gray of a transform (mode 0 linear / 1 sqrt_linear): 0, or 1 when the
// reference throws (no finite value).
int dfref_transform_gray(const std::uint8_t* img, std::size_t rows, std::size_t cols, int metric, int mode,
                         std::uint8_t* out) {
    try {
        const auto g = to_gray(ref_transform(to_image(img, rows, cols), metric),
                               mode ? GrayMapping::sqrt_linear : GrayMapping::linear);
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t j = 0; j < cols; ++j) out[i * cols + j] = g(i, j);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// labels_to_gray(voronoi_labels(img), object_count) and to_text(labels):
// 0, or 1 when the reference throws (no features).
int dfref_labels_render(const std::uint8_t* img, std::size_t rows, std::size_t cols, std::uint8_t* gray, char* text,
                        std::size_t cap, int* text_len) {
    try {
        const auto bi = to_image(img, rows, cols);
        const auto lab = voronoi_labels(bi);
        const auto g = labels_to_gray(lab, bi.object_count());
        for (std::size_t i = 0; i < rows; ++i)
            for (std::size_t j = 0; j < cols; ++j) gray[i * cols + j] = g(i, j);
        *text_len = put_text(to_text(lab), text, cap);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// danielsson(img) / danielsson_first_sweep(img) (vector_dt.cpp:108-124): the
// squared-distance map and the offset components (Offset::kUnset where unset).
int dfref_danielsson(const std::uint8_t* img, std::size_t rows, std::size_t cols, int first_only, std::uint64_t* dist,
                     std::uint32_t* dy, std::uint32_t* dx) {
    const auto bi = to_image(img, rows, cols);
    const auto r = first_only ? danielsson_first_sweep(bi) : danielsson(bi);
    copy_map(r.distance, dist);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) {
            dy[i * cols + j] = r.offsets(i, j).dy;
            dx[i * cols + j] = r.offsets(i, j).dx;
        }
    return 0;
}

std::uint64_t dfref_kind_bound(int kind, std::size_t rows, std::size_t cols) {
    return kind_bound(static_cast<DistanceKind>(kind), rows, cols);
}

}  // extern "C"
