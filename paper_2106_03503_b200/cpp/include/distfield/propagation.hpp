// distfield/propagation.hpp -- drop-in for the reference's propagation
// transforms (/root/reference/proj/core/include/distfield/propagation.hpp),
// computed on the GPU: the whole transforms from the separable closed forms
// (bit-exact with the two-pass raster scans, SURVEY.md finding 6); the
// per-pass in-place functions (:15-26) by dfc_raster_pass_u64 over the
// caller's map (k_passes.cu: the reference's relaxation order, rows in
// sequence, the chain along a row as a scan).
#pragma once

#include "distfield/grid.hpp"

namespace distfield {

// In-place passes over a map (init_distance_map or any other), as the
// reference: propagation.hpp:15-26.  `threads` is accepted and ignored.
void cityblock_forward_pass(DistanceMap& dm);
void cityblock_backward_pass(DistanceMap& dm);
void cityblock_vertical_passes(DistanceMap& dm, unsigned threads = 1);
void cityblock_horizontal_passes(DistanceMap& dm, unsigned threads = 1);
void chamfer_forward_pass(DistanceMap& dm);
void chamfer_backward_pass(DistanceMap& dm);

DistanceMap cityblock_sequential(const BinaryImage& img);
DistanceMap cityblock_separable(const BinaryImage& img, unsigned threads = 1);
DistanceMap chamfer34(const BinaryImage& img);

// B200 addition: the chessboard (L-infinity) transform the paper compares
// against; the reference only has a brute-force test oracle
// (proj/tests/oracles.hpp:52-55).  kind() == DistanceKind::chessboard.
DistanceMap chessboard(const BinaryImage& img);

// (d / 3)^2 per cell of a chamfer-3-4 map (propagation.cpp:111-127);
// std::invalid_argument for any other kind.
Grid<double> chamfer_normalized(const DistanceMap& dm);

}  // namespace distfield
