// dfc_all.cu -- the single translation unit of libdfc.so: every kernel and
// the C ABI are compiled together (whole-program, no relocatable device
// code), so kernel host stubs, templates and registrations live in one unit.
#include "k_columns.cu"
#include "k_rows.cu"
#include "k_rows_dense.cu"
#include "k_rows_lr.cu"
#include "k_rows_pts.cu"
#include "k_rows_band.cu"
#include "k_rows_anc.cu"
#include "k_raster.cu"
#include "k_raster_anc.cu"
#include "k_render.cu"
#include "k_passes.cu"
#include "k_vector.cu"
#include "dfc_api.cu"
#include "dfc_shard.cu"
