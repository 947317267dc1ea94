/*
 * oracle/dt_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference `distfield` hot path
 * (/root/reference/proj/core/src/{grid,exact_edt,propagation,random_image}.cpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product path (paper_2106_03503_b200/) never does.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (1) the reference's own golden matrices (proj/tests/goldens.hpp, dumped to
 *       tests/golden/six_point.json by tests/golden/make_golden.py), and
 *   (2) the reference itself compiled from its sources into oracle/_ref/
 *       (oracle/Makefile + oracle/ref_shim.cpp) on seeded random images.
 *
 * Conventions follow the reference: row-major cells, object = nonzero byte
 * (grid.hpp:82), distances as uint64 with UINT64_MAX as the infinity marker
 * (grid.hpp:113), labels as uint32 feature ordinals with UINT32_MAX = none
 * (grid.hpp:174).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF UINT64_MAX
#define ORC_NOCOL UINT32_MAX

enum { ORC_CITYBLOCK = 0, ORC_CHESSBOARD = 1, ORC_CHAMFER3 = 2, ORC_SQEUCLID = 3 };

/* kind_bound -- grid.cpp:54-64 */
uint64_t orc_kind_bound(int kind, uint64_t rows, uint64_t cols) {
    const uint64_t dr = rows - 1, dc = cols - 1;
    switch (kind) {
        case ORC_CITYBLOCK: return dr + dc;
        case ORC_CHESSBOARD: return dr > dc ? dr : dc;
        case ORC_CHAMFER3: return 4 * (dr + dc);
        default: return dr * dr + dc * dc;
    }
}

/* Xorshift64Star -- random_image.hpp:12-29 */
typedef struct { uint64_t s; } orc_rng;
static void rng_seed(orc_rng* r, uint64_t seed) { r->s = seed ? seed : 0x9e3779b97f4a7c15ULL; }
static uint64_t rng_next(orc_rng* r) {
    r->s ^= r->s >> 12;
    r->s ^= r->s << 25;
    r->s ^= r->s >> 27;
    return r->s * 0x2545f4914f6cdd1dULL;
}
static double rng_unit(orc_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

/* generate_random_image -- random_image.cpp:5-15 (row-major Bernoulli draws) */
void orc_generate_random_image(uint64_t rows, uint64_t cols, double density, uint64_t seed,
                               uint8_t* out) {
    orc_rng r;
    rng_seed(&r, seed);
    for (uint64_t p = 0; p < rows * cols; ++p) out[p] = rng_unit(&r) < density ? 1 : 0;
}

/* init_distance_map -- grid.cpp:85-91 */
void orc_init_map(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t* dm) {
    for (uint64_t p = 0; p < rows * cols; ++p) dm[p] = img[p] ? 0 : ORC_INF;
}

/* vertical_down_pass -- exact_edt.cpp:74-91 (odd-step increments, strict '>') */
void orc_vertical_down_pass(uint64_t* dm, uint64_t rows, uint64_t cols) {
    for (uint64_t j = 0; j < cols; ++j) {
        uint64_t step = 1;
        for (uint64_t i = 1; i < rows; ++i) {
            const uint64_t above = dm[(i - 1) * cols + j];
            uint64_t* cell = &dm[i * cols + j];
            if (above != ORC_INF && (*cell == ORC_INF || *cell > above + step)) {
                *cell = above + step;
                step += 2;
            } else {
                step = 1;
            }
        }
    }
}

/* vertical_up_pass -- exact_edt.cpp:93-110 */
void orc_vertical_up_pass(uint64_t* dm, uint64_t rows, uint64_t cols) {
    for (uint64_t j = 0; j < cols; ++j) {
        uint64_t step = 1;
        for (uint64_t i = rows - 1; i-- > 0;) {
            const uint64_t below = dm[(i + 1) * cols + j];
            uint64_t* cell = &dm[i * cols + j];
            if (below != ORC_INF && (*cell == ORC_INF || *cell > below + step)) {
                *cell = below + step;
                step += 2;
            } else {
                step = 1;
            }
        }
    }
}

/* vertical_pass -- exact_edt.cpp:112-117 */
void orc_vertical_pass(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t* dm) {
    orc_init_map(img, rows, cols, dm);
    orc_vertical_down_pass(dm, rows, cols);
    orc_vertical_up_pass(dm, rows, cols);
}

/* ceil_div / floor_div -- exact_edt.cpp:17-27 (den > 0) */
static int64_t ceil_div(int64_t num, int64_t den) {
    int64_t q = num / den;
    if (num % den > 0) ++q;
    return q;
}
static int64_t floor_div(int64_t num, int64_t den) {
    int64_t q = num / den;
    if (num % den != 0 && num < 0) --q;
    return q;
}

/* local_max -- exact_edt.cpp:13-15 */
static int64_t local_max(uint64_t rows, uint64_t cols) {
    return (int64_t)orc_kind_bound(ORC_SQEUCLID, rows, cols) + 1;
}

/*
 * build_row_envelope -- exact_edt.cpp:190-230.
 * vert: one row, sentinel-substituted (>= lmax means "no feature in column").
 * ks must hold cols+1 entries, js cols+2. Returns the number of ks entries;
 * js has one more. *evals accumulates the boundary evaluations (:199-201).
 */
int64_t orc_build_row_envelope(const int64_t* vert, int64_t cols, int64_t lmax, int take_new,
                               int64_t* ks, int64_t* js, uint64_t* evals) {
    uint64_t ev = 0;
#define BOUNDARY(k, m)                                                              \
    (++ev, take_new ? ceil_div(vert[(m)] - vert[(k)] - (k) * (k) + (m) * (m), 2 * ((m) - (k))) \
                    : floor_div(vert[(m)] - vert[(k)] - (k) * (k) + (m) * (m), 2 * ((m) - (k))) + 1)
    int64_t idx = 0;
    js[0] = -lmax;
    ks[0] = 0;
    for (int64_t m = 1; m < cols; ++m) {
        if (vert[m] >= lmax) continue;
        int64_t start = BOUNDARY(ks[idx], m);
        while (start <= js[idx]) {
            --idx;
            start = BOUNDARY(ks[idx], m);
        }
        if (start <= cols - 1) {
            ++idx;
            js[idx] = start > 0 ? start : 0;
            ks[idx] = m;
        }
    }
#undef BOUNDARY
    js[0] = 0;
    js[idx + 1] = cols;
    if (evals) *evals += ev;
    return idx + 1;
}

/*
 * envelope_rows + meijster_scan -- exact_edt.cpp:242-283.
 * take_new = 1 reproduces meijster_scan (nearest_col = largest minimizing
 * column); take_new = 0 is the keep_old policy used by voronoi_labels
 * (:363). out: squared distances (INF where the serving vertex is a sentinel,
 * store_value :38-41). nearest_col may be NULL.
 */
void orc_envelope_scan(const uint64_t* vert, uint64_t rows, uint64_t cols, int take_new,
                       uint64_t* out, uint32_t* nearest_col, uint64_t* candidates) {
    const int64_t lmax = local_max(rows, cols);
    int64_t* buf = (int64_t*)malloc(sizeof(int64_t) * cols);
    int64_t* ks = (int64_t*)malloc(sizeof(int64_t) * (cols + 1));
    int64_t* js = (int64_t*)malloc(sizeof(int64_t) * (cols + 2));
    uint64_t cand = 0;
    for (uint64_t i = 0; i < rows; ++i) {
        for (uint64_t j = 0; j < cols; ++j) {  /* load_row :29-35 */
            const uint64_t v = vert[i * cols + j];
            buf[j] = v == ORC_INF ? lmax : (int64_t)v;
        }
        const int64_t n = orc_build_row_envelope(buf, (int64_t)cols, lmax, take_new, ks, js, &cand);
        for (int64_t t = 0; t < n; ++t) {
            const int64_t k = ks[t], vk = buf[k];
            for (int64_t j = js[t]; j < js[t + 1]; ++j) {
                const int64_t d = vk + (j - k) * (j - k);
                ++cand;
                out[i * cols + j] = d >= lmax ? ORC_INF : (uint64_t)d;
                if (nearest_col) nearest_col[i * cols + j] = vk >= lmax ? ORC_NOCOL : (uint32_t)k;
            }
        }
    }
    free(buf);
    free(ks);
    free(js);
    if (candidates) *candidates += cand;
}

/* edt(img, envelope) -- exact_edt.cpp:285-317 (envelope path, no transpose) */
void orc_edt(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t* out) {
    uint64_t* vert = (uint64_t*)malloc(sizeof(uint64_t) * rows * cols);
    orc_vertical_pass(img, rows, cols, vert);
    orc_envelope_scan(vert, rows, cols, 1, out, NULL, NULL);
    free(vert);
}

/*
 * voronoi_labels -- exact_edt.cpp:319-371. labels = feature ordinals
 * (row-major enumeration, grid.cpp:29-36). Returns -1 (the reference throws
 * std::domain_error, :321) when the image has no object pixel.
 * If linear != NULL it additionally receives row*cols+col of each label.
 */
int orc_voronoi_labels(const uint8_t* img, uint64_t rows, uint64_t cols, uint32_t* labels,
                       int32_t* linear) {
    const uint64_t n = rows * cols;
    uint32_t* id_at = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t id = 0;
    for (uint64_t p = 0; p < n; ++p) id_at[p] = img[p] ? id++ : ORC_NOCOL;
    if (id == 0) {
        free(id_at);
        return -1;
    }
    uint64_t* vert = (uint64_t*)malloc(sizeof(uint64_t) * n);
    uint32_t* src_row = (uint32_t*)malloc(sizeof(uint32_t) * n);
    orc_init_map(img, rows, cols, vert);
    for (uint64_t p = 0; p < n; ++p) src_row[p] = ORC_NOCOL;
    for (uint64_t j = 0; j < cols; ++j) {  /* fused vertical pass :331-360 */
        for (uint64_t i = 0; i < rows; ++i)
            if (img[i * cols + j]) src_row[i * cols + j] = (uint32_t)i;
        uint64_t step = 1;
        for (uint64_t i = 1; i < rows; ++i) {
            const uint64_t above = vert[(i - 1) * cols + j];
            uint64_t* cell = &vert[i * cols + j];
            if (above != ORC_INF && (*cell == ORC_INF || *cell > above + step)) {
                *cell = above + step;
                src_row[i * cols + j] = src_row[(i - 1) * cols + j];
                step += 2;
            } else {
                step = 1;
            }
        }
        step = 1;
        for (uint64_t i = rows - 1; i-- > 0;) {
            const uint64_t below = vert[(i + 1) * cols + j];
            uint64_t* cell = &vert[i * cols + j];
            if (below != ORC_INF && (*cell == ORC_INF || *cell > below + step)) {
                *cell = below + step;
                src_row[i * cols + j] = src_row[(i + 1) * cols + j];
                step += 2;
            } else {
                step = 1;
            }
        }
    }
    /* envelope_rows(keep_old) :362-369 */
    uint64_t* dist = (uint64_t*)malloc(sizeof(uint64_t) * n);
    uint32_t* col = (uint32_t*)malloc(sizeof(uint32_t) * n);
    orc_envelope_scan(vert, rows, cols, 0, dist, col, NULL);
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
            const uint32_t k = col[i * cols + j];
            uint32_t lab = ORC_NOCOL;
            int32_t lin = -1;
            if (k != ORC_NOCOL) {
                const uint64_t r = src_row[i * cols + k];
                lab = id_at[r * cols + k];
                lin = (int32_t)(r * cols + k);
            }
            labels[i * cols + j] = lab;
            if (linear) linear[i * cols + j] = lin;
        }
    free(id_at);
    free(vert);
    free(src_row);
    free(dist);
    free(col);
    return 0;
}

/* relax -- propagation.cpp:10-12 */
static inline void relax(uint64_t* cell, uint64_t nbr, uint64_t w) {
    if (nbr != ORC_INF && *cell > nbr + w) *cell = nbr + w;
}

/* cityblock_forward_pass / _backward_pass / cityblock_sequential -- propagation.cpp:16-34, 90-95 */
void orc_cityblock_sequential(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t* dm) {
    orc_init_map(img, rows, cols, dm);
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
            if (i > 0) relax(&dm[i * cols + j], dm[(i - 1) * cols + j], 1);
            if (j > 0) relax(&dm[i * cols + j], dm[i * cols + j - 1], 1);
        }
    for (uint64_t i = rows; i-- > 0;)
        for (uint64_t j = cols; j-- > 0;) {
            if (i + 1 < rows) relax(&dm[i * cols + j], dm[(i + 1) * cols + j], 1);
            if (j + 1 < cols) relax(&dm[i * cols + j], dm[i * cols + j + 1], 1);
        }
}

/*
 * Two 8-neighbour raster passes with axis weight `wa` and diagonal weight
 * `wd`, in the exact visiting order of chamfer_forward_pass /
 * chamfer_backward_pass (propagation.cpp:60-88).
 *  wa=3, wd=4: chamfer34 (propagation.cpp:104-109).
 *  wa=1, wd=1: chessboard -- NO reference transform exists; this builder
 *              restatement is pinned to oracle::chessboard
 *              (proj/tests/oracles.hpp:52-55) by tests/test_oracle.py.
 */
void orc_raster8(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t wa, uint64_t wd,
                 uint64_t* dm) {
    orc_init_map(img, rows, cols, dm);
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
            uint64_t* cell = &dm[i * cols + j];
            if (j > 0) relax(cell, dm[i * cols + j - 1], wa);
            if (i > 0) {
                relax(cell, dm[(i - 1) * cols + j], wa);
                if (j > 0) relax(cell, dm[(i - 1) * cols + j - 1], wd);
                if (j + 1 < cols) relax(cell, dm[(i - 1) * cols + j + 1], wd);
            }
        }
    for (uint64_t i = rows; i-- > 0;)
        for (uint64_t j = cols; j-- > 0;) {
            uint64_t* cell = &dm[i * cols + j];
            if (j + 1 < cols) relax(cell, dm[i * cols + j + 1], wa);
            if (i + 1 < rows) {
                relax(cell, dm[(i + 1) * cols + j], wa);
                if (j > 0) relax(cell, dm[(i + 1) * cols + j - 1], wd);
                if (j + 1 < cols) relax(cell, dm[(i + 1) * cols + j + 1], wd);
            }
        }
}

/*
 * The per-pass in-place functions over any uint64 map, in the reference's
 * visiting order -- propagation.cpp:16-88.  pass: 0 cityblock_forward_pass
 * (:16-24), 1 cityblock_backward_pass (:26-34), 2 cityblock_vertical_passes
 * (:36-46), 3 cityblock_horizontal_passes (:48-58), 4 chamfer_forward_pass
 * (:60-73), 5 chamfer_backward_pass (:75-88).
 */
void orc_raster_pass(uint64_t* dm, uint64_t rows, uint64_t cols, int pass) {
    if (pass == 0) {
        for (uint64_t i = 0; i < rows; ++i)
            for (uint64_t j = 0; j < cols; ++j) {
                if (i > 0) relax(&dm[i * cols + j], dm[(i - 1) * cols + j], 1);
                if (j > 0) relax(&dm[i * cols + j], dm[i * cols + j - 1], 1);
            }
    } else if (pass == 1) {
        for (uint64_t i = rows; i-- > 0;)
            for (uint64_t j = cols; j-- > 0;) {
                if (i + 1 < rows) relax(&dm[i * cols + j], dm[(i + 1) * cols + j], 1);
                if (j + 1 < cols) relax(&dm[i * cols + j], dm[i * cols + j + 1], 1);
            }
    } else if (pass == 2) {
        for (uint64_t j = 0; j < cols; ++j) {
            for (uint64_t i = 1; i < rows; ++i) relax(&dm[i * cols + j], dm[(i - 1) * cols + j], 1);
            for (uint64_t i = rows - 1; i-- > 0;) relax(&dm[i * cols + j], dm[(i + 1) * cols + j], 1);
        }
    } else if (pass == 3) {
        for (uint64_t i = 0; i < rows; ++i) {
            for (uint64_t j = 1; j < cols; ++j) relax(&dm[i * cols + j], dm[i * cols + j - 1], 1);
            for (uint64_t j = cols - 1; j-- > 0;) relax(&dm[i * cols + j], dm[i * cols + j + 1], 1);
        }
    } else if (pass == 4) {
        for (uint64_t i = 0; i < rows; ++i)
            for (uint64_t j = 0; j < cols; ++j) {
                uint64_t* cell = &dm[i * cols + j];
                if (j > 0) relax(cell, dm[i * cols + j - 1], 3);
                if (i > 0) {
                    relax(cell, dm[(i - 1) * cols + j], 3);
                    if (j > 0) relax(cell, dm[(i - 1) * cols + j - 1], 4);
                    if (j + 1 < cols) relax(cell, dm[(i - 1) * cols + j + 1], 4);
                }
            }
    } else if (pass == 5) {
        for (uint64_t i = rows; i-- > 0;)
            for (uint64_t j = cols; j-- > 0;) {
                uint64_t* cell = &dm[i * cols + j];
                if (j + 1 < cols) relax(cell, dm[i * cols + j + 1], 3);
                if (i + 1 < rows) {
                    relax(cell, dm[(i + 1) * cols + j], 3);
                    if (j > 0) relax(cell, dm[(i + 1) * cols + j - 1], 4);
                    if (j + 1 < cols) relax(cell, dm[(i + 1) * cols + j + 1], 4);
                }
            }
    }
}

void orc_chamfer34(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t* dm) {
    orc_raster8(img, rows, cols, 3, 4, dm);
}
void orc_chessboard(const uint8_t* img, uint64_t rows, uint64_t cols, uint64_t* dm) {
    orc_raster8(img, rows, cols, 1, 1, dm);
}

/*
 * Brute-force minimum over features -- proj/tests/oracles.hpp:28-55, 56-59.
 * metric: 0 city-block (a+b), 1 chessboard max(a,b), 3 squared euclidean.
 */
void orc_brute(const uint8_t* img, uint64_t rows, uint64_t cols, int metric, uint64_t* dm) {
    uint64_t nf = 0;
    for (uint64_t p = 0; p < rows * cols; ++p) nf += img[p] != 0;
    uint64_t* fr = (uint64_t*)malloc(sizeof(uint64_t) * (nf + 1));
    uint64_t* fc = (uint64_t*)malloc(sizeof(uint64_t) * (nf + 1));
    nf = 0;
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j)
            if (img[i * cols + j]) {
                fr[nf] = i;
                fc[nf] = j;
                ++nf;
            }
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
            uint64_t best = ORC_INF;
            for (uint64_t f = 0; f < nf; ++f) {
                const uint64_t a = i > fr[f] ? i - fr[f] : fr[f] - i;
                const uint64_t b = j > fc[f] ? j - fc[f] : fc[f] - j;
                const uint64_t d = metric == 0 ? a + b : metric == 1 ? (a > b ? a : b) : a * a + b * b;
                if (d < best) best = d;
            }
            dm[i * cols + j] = best;
        }
    free(fr);
    free(fc);
}

/* ---- Danielsson vector transform (vector_dt.cpp:41-116) ----
 * Offsets are magnitudes (dy, dx), ORC_UNSET where no feature was claimed yet
 * (vector_dt.hpp:15-19); a cell is overwritten only on a strictly smaller
 * squared distance (:58).  sweep_down (:64-79): per row, the vertical update,
 * then left-to-right (from the left neighbour, then from the upper-left one),
 * then right-to-left (from the upper-right one, then from the right
 * neighbour).  sweep_up (:81-96) mirrors it with the row below, the in-row
 * neighbour first in BOTH of its horizontal passes.  first_only = 1 is
 * danielsson_first_sweep (:118-124). */
#define ORC_UNSET 0xFFFFFFFFu
static void dn_update(uint64_t* dist, uint32_t* dy, uint32_t* dx, uint64_t cols, uint64_t i, uint64_t j,
                      uint64_t si, uint64_t sj, uint32_t ay, uint32_t ax) {
    const uint64_t s = si * cols + sj, p = i * cols + j;
    if (dy[s] == ORC_UNSET) return; /* :53 */
    const uint32_t ny = dy[s] + ay, nx = dx[s] + ax;
    const uint64_t d = (uint64_t)ny * ny + (uint64_t)nx * nx; /* :45-48 */
    if (dist[p] > d) { /* :58 strict */
        dist[p] = d;
        dy[p] = ny;
        dx[p] = nx;
    }
}

void orc_danielsson(const uint8_t* img, uint64_t rows, uint64_t cols, int first_only, uint64_t* dist,
                    uint32_t* dy, uint32_t* dx) {
    orc_init_map(img, rows, cols, dist); /* init_state :98-106 */
    for (uint64_t p = 0; p < rows * cols; ++p) dy[p] = dx[p] = img[p] ? 0u : ORC_UNSET;
    for (uint64_t i = 1; i < rows; ++i) { /* sweep_down :64-79 */
        for (uint64_t j = 0; j < cols; ++j) dn_update(dist, dy, dx, cols, i, j, i - 1, j, 1, 0);
        for (uint64_t j = 1; j < cols; ++j) {
            dn_update(dist, dy, dx, cols, i, j, i, j - 1, 0, 1);
            dn_update(dist, dy, dx, cols, i, j, i - 1, j - 1, 1, 1);
        }
        for (uint64_t j = cols - 1; j-- > 0;) {
            dn_update(dist, dy, dx, cols, i, j, i - 1, j + 1, 1, 1);
            dn_update(dist, dy, dx, cols, i, j, i, j + 1, 0, 1);
        }
    }
    if (first_only) return;
    for (uint64_t i = rows - 1; i-- > 0;) { /* sweep_up :81-96 */
        for (uint64_t j = 0; j < cols; ++j) dn_update(dist, dy, dx, cols, i, j, i + 1, j, 1, 0);
        for (uint64_t j = 1; j < cols; ++j) {
            dn_update(dist, dy, dx, cols, i, j, i, j - 1, 0, 1);
            dn_update(dist, dy, dx, cols, i, j, i + 1, j - 1, 1, 1);
        }
        for (uint64_t j = cols - 1; j-- > 0;) {
            dn_update(dist, dy, dx, cols, i, j, i, j + 1, 0, 1);
            dn_update(dist, dy, dx, cols, i, j, i + 1, j + 1, 1, 1);
        }
    }
}
