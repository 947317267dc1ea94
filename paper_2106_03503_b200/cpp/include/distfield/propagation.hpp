// distfield/propagation.hpp -- drop-in for the reference's propagation
// transforms (/root/reference/proj/core/include/distfield/propagation.hpp:28-30),
// computed on the GPU from the separable closed forms (bit-exact with the
// two-pass raster scans, SURVEY.md finding 6).  The per-pass in-place
// functions (cityblock_forward_pass, chamfer_backward_pass, ...) expose the
// intermediate states of the serial raster algorithm, which the GPU path does
// not have; they are not part of this drop-in.
#pragma once

#include "distfield/grid.hpp"

namespace distfield {

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
