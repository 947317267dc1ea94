/*
 * distfield_cuda.h -- the C ABI of the B200-native distance-transform hot path.
 *
 * This is the thin, never-throwing boundary the C++ drop-in library
 * (paper_2106_03503_b200/cpp, namespace distfield) and the Python host mirror
 * (paper_2106_03503_b200/__init__.py, via ctypes) call.  Plain pointers and
 * sizes only; all image/distance pointers are DEVICE pointers owned by the
 * caller; every call is stream-ordered on `stream` (0 = legacy default) with
 * no hidden host synchronisation.  Scratch comes from the device's default
 * stream-ordered memory pool (cudaMallocAsync / cudaFreeAsync).
 *
 * Conventions (reference: /root/reference/proj/core):
 *   - input: row-major uint8, object pixel = any nonzero byte (grid.hpp:82),
 *     rows of `pitch_bytes` bytes (>= cols);
 *   - outputs: dense row-major, row stride = cols elements;
 *   - squared distances int32; the reference's uint64 infinity marker
 *     (DistanceMap::kInfinity, grid.hpp:113) maps to DFC_INF_I32.  Infinity
 *     only occurs for an image without any object pixel (grid.hpp:109-110);
 *   - float distances: (float)sqrt((double)D) -- exactly the value the
 *     reference prints via to_text_sqrt (grid.cpp:146) -- and +inf for
 *     DFC_INF_I32;
 *   - labels: int32 LINEAR index row*cols+col of the nearest object pixel,
 *     ties broken exactly as voronoi_labels (exact_edt.cpp:319-371): the
 *     smallest minimising column, then the upper feature in that column.
 *     -1 for a featureless image (the reference throws std::domain_error,
 *     exact_edt.cpp:321; the C++ adapter rethrows);
 *   - nearest_col: meijster_scan().nearest_col (exact_edt.cpp:272-283): the
 *     LARGEST minimising column (take_new), -1 for kNoColumn.
 *   - supported shapes: 1 <= rows, cols <= 65535 and
 *     (rows-1)^2 + (cols-1)^2 <= DFC_MAX_SQDIST (the int32 result range;
 *     32768 x 32768 fits).  Larger shapes return DFC_ERR_SHAPE.
 */
#ifndef DISTFIELD_CUDA_H
#define DISTFIELD_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dfc_stream_t; /* == cudaStream_t */

#define DFC_INF_I32 0x7FFFFFFF
#define DFC_MAX_SQDIST 0x7FFFFFFE

enum dfc_status {
    DFC_OK = 0,
    DFC_ERR_SHAPE = 1,       /* rows/cols out of the supported range        */
    DFC_ERR_ARG = 2,         /* null/misaligned pointer, bad pitch or flag  */
    DFC_ERR_CUDA = 3,        /* a CUDA runtime error; see dfc_last_cuda_error */
    DFC_ERR_NCCL = 4,        /* multi-GPU exchange failed                   */
    DFC_ERR_NO_FEATURES = 5  /* label ordinals requested on a featureless image */
};

/* Polarity of the transform. BG_TO_OBJ is the reference `edt(img)`;
 * OBJ_TO_BG is `edt(img.inverted())` (grid.cpp:38-44, CLI --polarity inside). */
enum dfc_polarity { DFC_BG_TO_OBJ = 0, DFC_OBJ_TO_BG = 1 };

/*
 * Exact squared Euclidean distance transform of one image.
 * Replaces distfield::edt(img, EdtAlgorithm::envelope, ...)
 *   (exact_edt.hpp:100-102 / exact_edt.cpp:285-317) = vertical_pass
 *   (exact_edt.cpp:112-117) + meijster_scan(...).map (exact_edt.cpp:272-283);
 * with d_label != NULL also voronoi_labels (exact_edt.cpp:319-371), and with
 * d_nearest_col != NULL also meijster_scan().nearest_col.
 * d_sqdist is required; d_dist, d_label, d_nearest_col are optional (NULL).
 */
int dfc_edt_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
               int polarity, int32_t* d_sqdist, float* d_dist, int32_t* d_label,
               int32_t* d_nearest_col, dfc_stream_t stream);

/*
 * Both polarities from ONE read of the input (config 2): background-to-object
 * (= edt(img)) and object-to-background (= edt(img.inverted())).
 * Any of the four outputs may be NULL except the two squared maps.
 */
int dfc_edt_u8_dual(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                    int32_t* d_sqdist_bg, float* d_dist_bg, int32_t* d_sqdist_obj,
                    float* d_dist_obj, dfc_stream_t stream);

/*
 * A batch of n same-shape images (config 3), image b at
 * d_imgs + b*image_stride_bytes; outputs dense [n][rows][cols].
 * Labels are linear indices WITHIN each image (-1 for a featureless image).
 */
int dfc_edt_u8_batched(const uint8_t* d_imgs, int64_t n, int64_t rows, int64_t cols,
                       int64_t pitch_bytes, int64_t image_stride_bytes, int32_t* d_sqdist,
                       float* d_dist, int32_t* d_label, dfc_stream_t stream);

/*
 * The stage-one vertical pass alone (exact_edt.cpp:112-117): per column the
 * squared vertical distance to the nearest object pixel in that column,
 * DFC_INF_I32 for a featureless column.  Replaces distfield::vertical_pass.
 */
int dfc_vertical_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                    int32_t* d_vert, dfc_stream_t stream);

/*
 * The three approximate raster transforms of config 4, each bit-exact with
 * the reference two-pass raster scans: city-block = cityblock_sequential
 * (propagation.cpp:90-95), chamfer-3-4 = chamfer34 (propagation.cpp:104-109),
 * chessboard = oracle::chessboard (proj/tests/oracles.hpp:52-55; the
 * reference has no library transform for it).  Any output may be NULL.
 */
int dfc_raster_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                  int32_t* d_cityblock, int32_t* d_chessboard, int32_t* d_chamfer34,
                  dfc_stream_t stream);

/*
 * Converts linear-index labels to the reference's LabelMap ordinals (the
 * row-major enumeration index among object pixels, grid.cpp:29-36) with an
 * exclusive prefix count of object pixels.  d_ordinal may alias d_label.
 */
int dfc_label_ordinals(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                       const int32_t* d_label, uint32_t* d_ordinal, dfc_stream_t stream);

/*
 * Stage one alone as a uint16 nearest-object-row plane (0xFFFF = no object in
 * the column): d_nr[i*nr_pitch + j] = the row of the nearest object pixel in
 * column j (upper one on ties, exact_edt.cpp:327-360).  The building block of
 * the column-striped multi-GPU path (config 5).  nr_pitch % 4 == 0,
 * nr_pitch >= cols rounded up to 4, d_nr 8-byte aligned.
 */
int dfc_column_nr_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes, int polarity,
                     uint16_t* d_nr, int64_t nr_pitch, dfc_stream_t stream);

/*
 * The two directions of stage one separately, over an arbitrary squared-
 * distance map in place (uint64 cells, UINT64_MAX = infinity, row pitch in
 * elements): vertical_down_pass / vertical_up_pass (exact_edt.cpp:74-110),
 * including the odd-step increment chain, the strict '>' update and the
 * unsigned arithmetic of the reference.  down followed by up over
 * init_distance_map(img) is vertical_pass (:112-117).
 */
int dfc_vertical_down_pass_u64(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems,
                               dfc_stream_t stream);
int dfc_vertical_up_pass_u64(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems,
                             dfc_stream_t stream);

/*
 * Stage two alone from a nearest-row plane that may be split into column
 * tiles: element (i, j) at d_nr[(j / tile_cols) * tile_stride_elems +
 * i * tile_cols + j % tile_cols]; tile_cols >= cols means one row-major
 * plane of row stride tile_cols.  Local row i is global row row0 + i (the
 * values in d_nr are global rows).  Labels are global linear indices
 * (row * cols + col).  This is the row-stripe half of the config-5 exchange:
 * the N all-to-all blocks are read in place.  tile_cols even.
 */
int dfc_rows_from_nr_u16(const uint16_t* d_nr, int64_t rows, int64_t cols, int64_t row0, int64_t tile_cols,
                         int64_t tile_stride_elems, int take_new, int32_t* d_sqdist, float* d_dist,
                         int32_t* d_label, int32_t* d_nearest_col, dfc_stream_t stream);

/*
 * Stage two alone, from a vertical-DISTANCE plane: d_vdist[i*pitch_elems+k]
 * = a (the squared vertical value is a*a), 0xFFFF = no feature in column k.
 * Replaces meijster_scan(vert) (exact_edt.cpp:272-283) for vertical maps of
 * perfect squares -- every map vertical_pass produces.  take_new = 1 is
 * meijster_scan's tie rule (nearest_col = largest minimising column), 0 the
 * keep_old rule; squared distances are identical either way.
 * pitch_elems must be even and d_vdist 4-byte aligned.
 */
int dfc_envelope_vdist_u16(const uint16_t* d_vdist, int64_t rows, int64_t cols, int64_t pitch_elems,
                           int take_new, int32_t* d_sqdist, float* d_dist, int32_t* d_nearest_col,
                           dfc_stream_t stream);

/*
 * build_row_envelope / envelope_rows over ARBITRARY int64 vertical rows
 * (exact_edt.cpp:190-283; exact_edt.hpp:71-72): for each of `rows` rows of
 * `cols` values (row pitch in elements), the owner of every column j -- the
 * smallest (take_new = 0, keep_old) or largest (take_new = 1) minimiser of
 * vert[k] + (j - k)^2 over column 0 (the envelope's base, kept even when it is
 * a sentinel) and the columns with vert[k] < lmax -- into d_owner (int32,
 * rows x cols dense) and, if d_value != NULL, that minimum (int64; >= lmax
 * means the base sentinel owns the column: the reference stores kInfinity and
 * kNoColumn there).  The reference's (ks, js) are the runs of d_owner.
 */
int dfc_row_owners_i64(const int64_t* d_vert, int64_t rows, int64_t cols, int64_t pitch_elems, int64_t lmax,
                       int take_new, int32_t* d_owner, int64_t* d_value, dfc_stream_t stream);

/*
 * The reference's per-pass in-place raster functions (propagation.hpp:15-26)
 * over a uint64 map (UINT64_MAX = infinity, row pitch in elements), with the
 * reference's relaxation (an infinite neighbour never contributes,
 * propagation.cpp:10-12); values must stay below 2^62.
 */
enum dfc_raster_pass {
    DFC_PASS_CITYBLOCK_FORWARD = 0,   /* cityblock_forward_pass     propagation.cpp:16-24 */
    DFC_PASS_CITYBLOCK_BACKWARD = 1,  /* cityblock_backward_pass    :26-34 */
    DFC_PASS_CITYBLOCK_VERTICAL = 2,  /* cityblock_vertical_passes  :36-46 */
    DFC_PASS_CITYBLOCK_HORIZONTAL = 3,/* cityblock_horizontal_passes :48-58 */
    DFC_PASS_CHAMFER_FORWARD = 4,     /* chamfer_forward_pass       :60-73 */
    DFC_PASS_CHAMFER_BACKWARD = 5     /* chamfer_backward_pass      :75-88 */
};
int dfc_raster_pass_u64(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems, int pass,
                        dfc_stream_t stream);

/*
 * Danielsson's vector transform (vector_dt.hpp:56-72, vector_dt.cpp:41-124):
 * the approximate Euclidean transform that propagates offset magnitudes,
 * bit-exact with the reference's downward + upward sweeps (first_sweep_only
 * != 0: danielsson_first_sweep, the downward sweep alone).  Per image, dense
 * rows x cols outputs: d_dist the squared lengths (UINT64_MAX = infinity,
 * DistanceMap::kInfinity), d_dy / d_dx the offset components (0xFFFFFFFF =
 * Offset::kUnset).  A strict raster recurrence: one warp per image, parallel
 * over the images of a batch and over 32 cells of a row at a time (see
 * csrc/k_vector.cu).  n_images >= 1; image_stride_bytes is ignored for 1.
 */
int dfc_danielsson_u8(const uint8_t* d_img, int64_t n_images, int64_t rows, int64_t cols, int64_t pitch_bytes,
                      int64_t image_stride_bytes, int first_sweep_only, uint64_t* d_dist, uint32_t* d_dy,
                      uint32_t* d_dx, dfc_stream_t stream);

/*
 * Float distances of a squared-distance map: (float)sqrt((double)D) for each
 * of n int32 values (DFC_INF_I32 -> +inf) -- the row pass's own epilogue
 * (grid.cpp:146 semantics), e.g. for a map from dfc_vertical_u8.
 */
int dfc_sqrt_i32(const int32_t* d_sqdist, float* d_dist, int64_t n, dfc_stream_t stream);

/*
 * CLI / rendering epilogues (k_render.cu).  They replace host loops of the
 * reference's I/O layer so the CLI path stays on the device:
 *
 * dfc_unpack_pbm: a P4 raster -- `rows` rows of `row_bytes` = ceil(cols/8)
 * bytes, MSB first, bit 1 = object (read_netpbm, netpbm.cpp:81-95) -- into a
 * uint8 0/1 image of pitch `pitch_bytes` (>= cols); invert != 0 flips it
 * (BinaryImage::inverted, grid.cpp:38-44, the CLI's --polarity inside).
 */
int dfc_unpack_pbm(const uint8_t* d_bits, int64_t rows, int64_t cols, int64_t row_bytes, int invert,
                   uint8_t* d_img, int64_t pitch_bytes, dfc_stream_t stream);

/* uint8 image -> 0/1 (object = nonzero, grid.hpp:82), optionally inverted;
 * d_dst may alias d_src when the pitches are equal. */
int dfc_binarize_u8(const uint8_t* d_src, int64_t rows, int64_t cols, int64_t src_pitch, int invert,
                    uint8_t* d_dst, int64_t dst_pitch, dfc_stream_t stream);

/* Object pixels of an image (BinaryImage::object_count), ADDED to *d_count
 * (a device uint64 the caller zeroes). */
int dfc_count_objects_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                         uint64_t* d_count, dfc_stream_t stream);

/*
 * to_gray (grid.cpp:93-110) of n int32 values: round(255 * v / max) (mode 0,
 * GrayMapping::linear) or round(255 * sqrt(v) / sqrt(max)) (mode 1,
 * sqrt_linear), double arithmetic and lround as the reference; all zeros when
 * max == 0.  *d_max (device int32) receives the max finite value, -1 if there
 * is none -- the caller raises the reference's domain_error on -1 after its
 * own synchronisation.  d_scratch: one device uint32.
 */
int dfc_gray_i32(const int32_t* d_map, int64_t n, int mode, uint8_t* d_gray, int32_t* d_max,
                 uint32_t* d_scratch, dfc_stream_t stream);

/* labels_to_gray (grid.cpp:112-121): round(255 * ordinal / feature_count). */
int dfc_labels_gray(const uint32_t* d_ordinal, int64_t n, int64_t feature_count, uint8_t* d_gray,
                    dfc_stream_t stream);

/*
 * ONE image over `world` GPUs (config 5): column stripes
 * for the column pass, an all-to-all of the compact column-pass products
 * (per band of 32 rows and column: the 32-bit object mask and the nearest
 * object rows above / below the band -- 8 B per 32 pixels), row stripes for
 * the row pass.  Replaces the `parallel_for` fan-out of edt
 * (exact_edt.cpp:53-154, parallel.hpp:13-30) across devices; the result is
 * bit-identical to dfc_edt_u8 on the whole image.
 *
 * Rank r owns columns [dfc_shard_cols(cols, world, r)) of the input and rows
 * [dfc_shard_rows(rows, world, r)) of the output (row stripes are whole bands
 * of 32 rows).  Each dfc_shard describes one LOCAL rank; n_local may be 1
 * (one process per GPU: comm from dfc_comm_init_rank) up to world (one process
 * driving every GPU: comms from dfc_comm_init_all, or all comm NULL -- then
 * the exchange is stream-ordered peer copies inside this process, and every
 * rank must be local).  The exchange is NCCL grouped send/recv on each shard's
 * stream; NCCL (libnccl.so.2) is opened at the first call that needs it.
 * Returns DFC_ERR_NCCL (see dfc_last_nccl_error) when it is unavailable.
 */
typedef struct dfc_shard {
    int device;              /* CUDA device of this rank                          */
    int rank;                /* 0 .. world-1                                      */
    const uint8_t* d_img;    /* its column stripe: rows x ncols, row pitch below  */
    int64_t pitch_bytes;
    int32_t* d_sqdist;       /* its row stripe of the result: nrows x cols         */
    float* d_dist;           /* optional float distances of the row stripe          */
    int32_t* d_label;        /* optional labels (global linear index, keep_old)    */
    void* comm;              /* ncclComm_t, or NULL (in-process exchange)          */
    dfc_stream_t stream;
} dfc_shard;

int dfc_edt_u8_sharded(const dfc_shard* shards, int n_local, int world, int64_t rows, int64_t cols,
                       int polarity);
/* The partition: column stripe and row stripe of `rank`. */
int dfc_shard_cols(int64_t cols, int world, int rank, int64_t* col0, int64_t* ncols);
int dfc_shard_rows(int64_t rows, int world, int rank, int64_t* row0, int64_t* nrows);
/* Communicators: a 128-byte NCCL unique id (rank 0 makes it, the caller
 * broadcasts it), one rank's communicator on the CURRENT device, or one per
 * listed device for a single process; opaque ncclComm_t handles. */
int dfc_comm_unique_id(uint8_t* id128);
int dfc_comm_init_rank(void** comm, int world, int rank, const uint8_t* id128);
int dfc_comm_init_all(void** comms, int ndev, const int* devices);
int dfc_comm_destroy(void* comm);
/* The ncclResult_t behind the last DFC_ERR_NCCL on this thread. */
int dfc_last_nccl_error(void);

/*
 * Measurement hook (bench.py): cudaEvent_t handles recorded on the call's
 * stream by the next dfc_edt_u8* calls on this thread -- ev_col_begin before
 * the column pass, ev_row_begin between column and row pass, ev_row_end
 * after the row pass.  NULL disables a record.  Costs nothing when unset.
 */
int dfc_set_profile_events(void* ev_col_begin, void* ev_row_begin, void* ev_row_end);

/*
 * Stage-2 kernel selection for the calls of this thread: 0 = library
 * default, 1 = segment/merge kernel (k_rows) for every row, 4 = dense-row
 * kernel (k_rows_dense) for rows with only short runs between object pixels,
 * the lane-per-row chunk scan (k_rows_lr) for sparse planes and k_rows for
 * the rest, 5 = k_rows_lr for every row (k_rows as its overflow fallback),
 * 6 = the default: point planes by k_rows_pts, sparse planes of single
 * images by the band path (k_rows_band.cu), every other row by anchored
 * segments (k_rows_anc, rows up to 16384 columns; wider rows by k_rows).
 * Modes 2 and 3 (retired kernels) return DFC_ERR_ARG.  Results are identical
 * in every mode; this is a performance/testing knob.
 */
int dfc_set_row_kernel(int mode);

/* Columns per warp chunk of the lane-per-row kernel (mode 5) for calls on the
 * calling thread: a multiple of 32, 0 = default (DFC_LR_CHUNK, else as wide as ~4096 warps allow).
 * Results are identical; a performance/testing knob. */
int dfc_set_lr_chunk(int cols);

/* Smallest image (rows * cols) whose sparse planes take the band path
 * (k_rows_band.cu) in the default mode, for calls on the calling thread;
 * smaller sparse planes use the lane-per-row kernel.  0 = every size, negative
 * = the default (DFC_BAND_MIN_PX, else 2^24 + 1).  A performance / testing
 * knob: results are identical. */
int dfc_set_band_min_pixels(int64_t pixels);

/* Number of kernels the last successful call on this thread enqueued. */
int dfc_last_launch_count(void);
/* Debug: with DFC_DEBUG_GUARD=1 in the environment every scratch allocation
 * of the library carries canary zones on both sides and a poisoned interior;
 * this returns the number of canary bytes overwritten so far on the current
 * device (synchronises), or -1 when the mode is off.  The stand-in for
 * compute-sanitizer memcheck/initcheck where that tool cannot be run. */
long long dfc_debug_guard_violations(void);
/* Human-readable status; never NULL. */
const char* dfc_status_string(int status);
/* The cudaError_t behind the last DFC_ERR_CUDA on this thread (0 if none). */
int dfc_last_cuda_error(void);
/* Library version string, e.g. "distfield-b200 0.1 sm_100a". */
const char* dfc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DISTFIELD_CUDA_H */
