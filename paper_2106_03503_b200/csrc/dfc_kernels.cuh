// dfc_kernels.cuh -- argument blocks and declarations of every kernel.
#pragma once
#include "dfc_common.cuh"

namespace dfc {

// Stage 1 (k_columns.cu)
struct ColArgs {
    const uint8_t* img;
    int64_t pitch;       // bytes between rows
    int64_t img_stride;  // bytes between images
    int n_img, H, W;
    int Wp;              // padded row length (elements) of the uint16 planes
    int nb;              // bands per image
    int pol0, npol;      // first polarity and number of polarity slots (1 or 2)
    bool vec;            // 4-byte loads are legal (pitch, base aligned)
    // point planes (<= kPtsCap object pixels, default row pass): K1a lists their
    // object pixels, K1b/K1c skip them (k_rows_pts works from the list)
    uint32_t* pts;                           // [plane][kPtsCap] keys col << 16 | row, nullable
    const unsigned long long* pcounts;       // object pixels per plane (K1a), for the skip
    // band masks (bit r = row 32 b + r of the column is nonzero) [img][nb][Wp],
    // written by K1a when non-null and read by K1c instead of the image; with
    // skip_full, K1c writes no nearest-row plane for planes the row pass reads
    // from the bands (neither point nor sparse planes: k_rows_anc stages those
    // rows from masks + carries)
    uint32_t* bmask;
    bool skip_full;
    // the band path (k_rows_band.cu) takes the sparse planes: no nearest-row
    // plane for them either
    bool skip_sparse;
    // object-column bits per (plane, band) [slot][img][nb][ceil(W/32)], nullable:
    // bit k of word w = column 32 w + k holds an object pixel in the band (the
    // band path's hull filter, k_rows_band.cu)
    uint32_t* objcol;
};

// Stage 2 (k_rows.cu)
struct RowArgs {
    const uint16_t* nr;       // nearest object row per (row, column), kNoRow = none
    int64_t nr_img_stride;    // elements between images/slots
    int Wp;                   // elements between rows of nr (inside one column tile)
    int tile_cols;            // columns per tile of the nr plane (>= W: one tile)
    int64_t tile_stride;      // elements between consecutive column tiles
    int row0;                 // global row of local row 0 (row-striped shards)
    int H, W;
    int64_t total_rows;       // n_img * H
    int T, L, R;              // threads per row, columns per thread, rows per CTA
    int row_smem_words;       // 32-bit words of shared memory per row
    // outputs (nullable); image b's plane at base + b * stride (bytes)
    char* D;  int64_t sD;
    char* S;  int64_t sS;
    char* LB; int64_t sL;
    char* NC; int64_t sN;
    bool vec;                 // 16-byte vector stores are legal
    bool vec_nr;              // 16-byte nr loads of a whole segment are legal (window kernel)
    bool vdist;               // nr holds vertical DISTANCES a (g = a^2), not rows
    const int* row_list;      // fallback mode: process only these rows (nullptr: all)
    const int* row_count;     // number of entries in row_list (device)
    uint8_t* row_done;        // per row: 1 = written by k_rows_dense, 2 = k_rows_lr overflowed
    bool lr_gate;             // rows of sparse planes belong to k_rows_lr (unless row_done == 2)
    bool pts_gate;            // rows of point planes belong to k_rows_pts
    const unsigned long long* plane_counts;  // object pixels per plane (dense gate), nullable
    // band source (k_rows_anc, nullable bmask = read nr): the column pass's band
    // masks [img][nb][Wp] and carries (nearest object row above / below each
    // band) [plane][nb][Wp]; plane p of this call is polarity bpol0 + p / n_img
    const uint32_t* bmask;
    const uint16_t* babove;
    const uint16_t* bbelow;
    int nb, n_img, bpol0;
};

// Raster transforms (k_raster.cu)
struct RasterArgs {
    const uint16_t* nr;
    int Wp, H, W;
    int T, L;
    int32_t* city;
    int32_t* chess;
    int32_t* cham;
    // band source (k_raster_anc; nullable bmask = read nr): K1a's masks and
    // K1b's carries above / below, [nb][Wp]
    const uint32_t* bmask;
    const uint16_t* babove;
    const uint16_t* bbelow;
};

// Point plane: at most kPtsCap object pixels (C3's 30-point images).  With
// the points path on (default row pass, rows per plane a multiple of 32) its
// rows go to k_rows_pts, which works from K1a's list of object pixels; no
// nearest-row plane is written or read for it.
constexpr int kPtsCap = 32;
__host__ __device__ __forceinline__ bool pts_plane(const unsigned long long* counts, int img, bool on) {
    return on && counts != nullptr && counts[img] <= (unsigned long long)kPtsCap;
}

// Sparse plane (object pixels < 1/c_sparse_div of the plane): its rows go to
// the band path (k_rows_band.cu) or the lane-per-row kernel (k_rows_lr.cu) in
// the default mode.  The divisor is a per-device constant (DFC_SPARSE_DIV,
// tuning; set once in init_pool_once).
__device__ __constant__ unsigned long long c_sparse_div = 256ull;
__device__ __forceinline__ bool lr_plane(const unsigned long long* counts, int img, int H, int W) {
    return counts != nullptr && counts[img] * c_sparse_div < (unsigned long long)H * (unsigned long long)W;
}

// Object mask of polarity `pol` (0: object = nonzero, 1: object = zero) from
// the nonzero mask m of a band with `valid` rows.
__host__ __device__ __forceinline__ uint32_t pol_mask(uint32_t m, int pol, uint32_t valid) {
    return pol ? (~m & valid) : m;
}

// The kernels themselves are defined in k_columns.cu / k_rows.cu / k_raster.cu and
// compiled in ONE translation unit with the C ABI (dfc_all.cu), so no
// forward declarations are needed (a declaration whose parameter qualifiers
// differ from the definition would name a different, undefined kernel).

}  // namespace dfc
