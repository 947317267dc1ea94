// distfield/exact_edt.hpp -- drop-in for the reference's exact EDT entry points
// (/root/reference/proj/core/include/distfield/exact_edt.hpp), computed on the
// GPU through the C ABI (include/distfield_cuda.h).  Same names, signatures,
// return types, tie rules and exceptions.  Every algorithm/orientation yields
// the identical map in the reference (exact_edt.hpp:97-99), so all are served
// by the GPU envelope path; `threads` is accepted and ignored.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "distfield/grid.hpp"

namespace distfield {

struct CostEstimate {
    std::uint64_t objects = 0;
    std::uint64_t background = 0;
    std::uint64_t computations = 0;
};

// Candidate counter.  The GPU path reports one evaluation per output cell
// (a deterministic, linear count; the reference's own value is algorithm
// internal, exact_edt.cpp:199-201/:260).
struct ScanStats {
    std::uint64_t candidates = 0;
};

struct EnvelopeState {
    std::vector<std::int64_t> ks;
    std::vector<std::int64_t> js;
};

enum class EnvelopeTie : std::uint8_t { take_new, keep_old };

constexpr std::uint32_t kNoColumn = std::numeric_limits<std::uint32_t>::max();

struct MeijsterResult {
    DistanceMap map;
    Grid<std::uint32_t> nearest_col;
};

enum class EdtAlgorithm : std::uint8_t { bruteforce, simple, improved, envelope };
enum class Orientation : std::uint8_t { automatic, rows, columns };

// Stage one: per column, the squared vertical distance to the nearest object.
// The two directions in place over any squared-distance map (exact_edt.cpp:74-110).
void vertical_down_pass(DistanceMap& dm, unsigned threads = 1);
void vertical_up_pass(DistanceMap& dm, unsigned threads = 1);
DistanceMap vertical_pass(const BinaryImage& img, unsigned threads = 1);

// Stage two over a vertical map (meijster_scan, take_new ties: nearest_col is
// the LARGEST minimising column).  Vertical-pass maps (every finite value a
// perfect square) take the uint16 vertical-distance path; any other map the
// generic int64 row-envelope kernel (dfc_row_owners_i64).
MeijsterResult meijster_scan(const DistanceMap& vert, ScanStats* stats = nullptr, unsigned threads = 1);

// build_row_envelope (exact_edt.hpp:71-72, exact_edt.cpp:190-230): the lower
// envelope of one row of int64 vertical values (entries >= local_max are
// sentinels, column 0 is always the base), computed on the device
// (dfc_row_owners_i64: the owner of every column under `tie`) and returned as
// the reference's (ks, js).  ScanStats counts one evaluation per column.
EnvelopeState build_row_envelope(std::span<const std::int64_t> vert, std::int64_t local_max, EnvelopeTie tie,
                                 ScanStats* stats = nullptr);

// Envelope bookkeeping of one row (take_new), rebuilt from the GPU's
// nearest-column row: ks = vertex columns (ks[0] = 0 base), js = segment
// starts with js.front() = 0, js.back() = cols.
EnvelopeState meijster_row_envelope(const DistanceMap& vert, std::size_t row);

// Exact squared euclidean transform.
DistanceMap edt(const BinaryImage& img, EdtAlgorithm algorithm, Orientation orient = Orientation::automatic,
                ScanStats* stats = nullptr, unsigned threads = 1);

// Voronoi labels (feature ordinals): smallest minimising column, then the
// upper feature.  Throws std::domain_error for an image without features.
LabelMap voronoi_labels(const BinaryImage& img, unsigned threads = 1);

// ---- B200 additions (no reference counterpart) ----
// Both polarities from one upload/read: {edt(img), edt(img.inverted())}.
std::pair<DistanceMap, DistanceMap> edt_both_polarities(const BinaryImage& img);
// Float distances (float)sqrt((double)D), +inf where D is infinite.
std::vector<float> edt_distances(const BinaryImage& img);

}  // namespace distfield
