/*
 * gen.c -- seeded synthetic inputs for the five BASELINE.json configs.
 *
 * The paper's figure images (cup, 30-point Voronoi, blob/hand) are not in the
 * reference tree (SURVEY.md finding 9); these generators are the stand-ins
 * specified in SURVEY.md section 8(d).  All randomness is the reference's own
 * xorshift64* (random_image.hpp:12-29) so the oracle and the GPU see
 * identical bytes.  Object pixels are 1, background 0.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s; } xs64;

static void xs_seed(xs64* r, uint64_t seed) { r->s = seed ? seed : 0x9e3779b97f4a7c15ULL; }
static uint64_t xs_next(xs64* r) {
    r->s ^= r->s >> 12;
    r->s ^= r->s << 25;
    r->s ^= r->s >> 27;
    return r->s * 0x2545f4914f6cdd1dULL;
}
static double xs_unit(xs64* r) { return (double)(xs_next(r) >> 11) * 0x1.0p-53; }

uint64_t dfg_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* C1: generate_random_image(rows, cols, density, seed) -- random_image.cpp:5-15 */
void dfg_bernoulli(uint8_t* out, int64_t rows, int64_t cols, double density, uint64_t seed) {
    xs64 r;
    xs_seed(&r, seed);
    for (int64_t p = 0; p < rows * cols; ++p) out[p] = xs_unit(&r) < density ? 1 : 0;
}

static void fill_disc(uint8_t* out, int64_t rows, int64_t cols, int64_t ci, int64_t cj, int64_t rad) {
    for (int64_t i = ci - rad; i <= ci + rad; ++i) {
        if (i < 0 || i >= rows) continue;
        const int64_t di = i - ci;
        for (int64_t j = cj - rad; j <= cj + rad; ++j) {
            if (j < 0 || j >= cols) continue;
            const int64_t dj = j - cj;
            if (di * di + dj * dj <= rad * rad) out[i * cols + j] = 1;
        }
    }
}

/* C2: n discs, centre uniform over the image, radius 8 + next()%57 (uniform in [8,64]) */
void dfg_discs(uint8_t* out, int64_t rows, int64_t cols, int64_t n, uint64_t seed) {
    xs64 r;
    xs_seed(&r, seed);
    memset(out, 0, (size_t)(rows * cols));
    for (int64_t t = 0; t < n; ++t) {
        const int64_t ci = (int64_t)(xs_next(&r) % (uint64_t)rows);
        const int64_t cj = (int64_t)(xs_next(&r) % (uint64_t)cols);
        const int64_t rad = 8 + (int64_t)(xs_next(&r) % 57);
        fill_disc(out, rows, cols, ci, cj, rad);
    }
}

/* C3: npts distinct points per image; image b uses seed splitmix64(master + b) */
void dfg_points_batch(uint8_t* out, int64_t nimg, int64_t rows, int64_t cols, int64_t npts,
                      uint64_t master) {
    memset(out, 0, (size_t)(nimg * rows * cols));
    for (int64_t b = 0; b < nimg; ++b) {
        xs64 r;
        xs_seed(&r, dfg_splitmix64(master + (uint64_t)b));
        uint8_t* img = out + b * rows * cols;
        int64_t placed = 0;
        while (placed < npts && placed < rows * cols) {
            const int64_t i = (int64_t)(xs_next(&r) % (uint64_t)rows);
            const int64_t j = (int64_t)(xs_next(&r) % (uint64_t)cols);
            if (img[i * cols + j]) continue; /* redraw duplicates */
            img[i * cols + j] = 1;
            ++placed;
        }
    }
}

/* C4: n shapes; type = next()&1; disc: d = 4 + next()%253, r = d/2, centre;
 * rectangle: h, w = 4 + next()%253, top-left corner; all clipped. */
void dfg_shapes(uint8_t* out, int64_t rows, int64_t cols, int64_t n, uint64_t seed) {
    xs64 r;
    xs_seed(&r, seed);
    memset(out, 0, (size_t)(rows * cols));
    for (int64_t t = 0; t < n; ++t) {
        if (xs_next(&r) & 1) {
            const int64_t d = 4 + (int64_t)(xs_next(&r) % 253);
            const int64_t ci = (int64_t)(xs_next(&r) % (uint64_t)rows);
            const int64_t cj = (int64_t)(xs_next(&r) % (uint64_t)cols);
            fill_disc(out, rows, cols, ci, cj, d / 2);
        } else {
            const int64_t h = 4 + (int64_t)(xs_next(&r) % 253);
            const int64_t w = 4 + (int64_t)(xs_next(&r) % 253);
            const int64_t i0 = (int64_t)(xs_next(&r) % (uint64_t)rows);
            const int64_t j0 = (int64_t)(xs_next(&r) % (uint64_t)cols);
            for (int64_t i = i0; i < i0 + h && i < rows; ++i)
                memset(out + i * cols + j0, 1, (size_t)((j0 + w < cols ? j0 + w : cols) - j0));
        }
    }
}

/* C5: the image is split into tile x tile tiles; ntiles_on of them (Fisher-Yates
 * over tile ids with next()%(t+1), first ntiles_on kept) receive Bernoulli(p)
 * object pixels, drawn in row-major pixel order only inside chosen tiles.
 * degenerate != 0: a single object pixel at (0, 0) instead. */
void dfg_sparse_tiles(uint8_t* out, int64_t rows, int64_t cols, int64_t tile, int64_t ntiles_on,
                      double p, uint64_t seed, int degenerate) {
    memset(out, 0, (size_t)(rows * cols));
    if (degenerate) {
        out[0] = 1;
        return;
    }
    xs64 r;
    xs_seed(&r, seed);
    const int64_t tr = (rows + tile - 1) / tile, tc = (cols + tile - 1) / tile, nt = tr * tc;
    int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)nt);
    uint8_t* on = (uint8_t*)calloc((size_t)nt, 1);
    for (int64_t t = 0; t < nt; ++t) ids[t] = t;
    for (int64_t t = nt - 1; t > 0; --t) {
        const int64_t k = (int64_t)(xs_next(&r) % (uint64_t)(t + 1));
        const int64_t tmp = ids[t];
        ids[t] = ids[k];
        ids[k] = tmp;
    }
    for (int64_t t = 0; t < ntiles_on && t < nt; ++t) on[ids[t]] = 1;
    for (int64_t i = 0; i < rows; ++i) {
        const uint8_t* onrow = on + (i / tile) * tc;
        uint8_t* row = out + i * cols;
        for (int64_t j0 = 0; j0 < cols; j0 += tile) {
            if (!onrow[j0 / tile]) continue;
            const int64_t j1 = j0 + tile < cols ? j0 + tile : cols;
            for (int64_t j = j0; j < j1; ++j) row[j] = xs_unit(&r) < p ? 1 : 0;
        }
    }
    free(ids);
    free(on);
}
