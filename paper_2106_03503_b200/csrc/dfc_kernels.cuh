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
};

// Stage 2 (k_rows.cu)
struct RowArgs {
    const uint16_t* nr;       // nearest object row per (row, column), kNoRow = none
    int64_t nr_img_stride;    // elements between images/slots
    int Wp;                   // elements between rows of nr
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
};

// Raster transforms (k_raster.cu)
struct RasterArgs {
    const uint16_t* nr;
    int Wp, H, W;
    int T, L;
    int32_t* city;
    int32_t* chess;
    int32_t* cham;
};

__global__ void k_band_summary(ColArgs a, uint16_t* first, uint16_t* last);
__global__ void k_band_scan(int W, int Wp, int nb, int64_t n_planes, uint16_t* first, uint16_t* last);
template <bool OUT_SQ>
__global__ void k_band_fill(ColArgs a, const uint16_t* below, const uint16_t* above, uint16_t* nr,
                            int32_t* vsq);
template <bool TAKE_NEW>
__global__ void k_rows(RowArgs a);
__global__ void k_raster(RasterArgs a);
__global__ void k_ord_rows(const uint8_t* img, int64_t pitch, int H, int W, int nw, uint32_t* masks,
                           uint32_t* wpre, uint32_t* rowcnt);
__global__ void k_ord_scan(const uint32_t* rowcnt, uint32_t* rowbase, int H);
__global__ void k_ord_map(const int32_t* label, int64_t n, int W, int nw, const uint32_t* masks,
                          const uint32_t* wpre, const uint32_t* rowbase, uint32_t* out);

}  // namespace dfc
