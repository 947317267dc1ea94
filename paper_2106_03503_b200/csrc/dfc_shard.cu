// dfc_shard.cu -- one giant image over N GPUs (config 5, north_star):
// column stripes for the column pass, an all-to-all of the COMPACT column-pass
// products, row stripes for the row pass.
//
//   1. rank g runs the column pass (K1a + K1b, k_columns.cu) on its column
//      stripe [col0_g, col1_g) -- exact, columns are independent: per band of
//      32 rows and column, the 32-bit object mask and the nearest object rows
//      above / below the band (global rows);
//   2. all-to-all: rank g sends rank q the bands of q's row stripe (a
//      contiguous band range, so three contiguous slices) and its object
//      count -- 8 B per (band, column) = 0.25 B/px instead of the 2 B/px of a
//      dense nearest-row plane (C5 at N = 8: 29 MB per GPU instead of 235 MB);
//      NCCL grouped send/recv (libnccl.so.2, opened at the first sharded call),
//      or, for shards of ONE process without communicators, stream-ordered
//      peer copies;
//   3. rank q repacks the N column tiles into full-width band rows and runs the
//      band path (k_rows_band.cu) on its row stripe: hull filter, per-row
//      stacks, fill, with global row numbers.  The band path is exact for any
//      plane (its density gate is only a performance choice), so every plane
//      takes it here and no host synchronisation is needed.
#include <dlfcn.h>
#include <nccl.h>

#include <functional>
#include <mutex>
#include <vector>

#include "dfc_kernels.cuh"

namespace {

using namespace dfc;

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

// NCCL is opened on first use: single-GPU callers never need it.  In a process
// that already holds libnccl.so.2 (torch) that copy is reused.
const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(sym("ncclCommInitAll"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommInitAll && a.CommDestroy && a.GroupStart && a.GroupEnd &&
               a.Send && a.Recv;
        return a;
    }();
    return api;
}

thread_local int g_last_nccl = 0;

int nccl_fail(ncclResult_t r) {
    g_last_nccl = (int)r;
    return DFC_ERR_NCCL;
}

void stripe_cols(int64_t cols, int world, int rank, int64_t& c0, int64_t& n) {
    c0 = cols * rank / world;
    n = cols * (rank + 1) / world - c0;
}

void stripe_bands(int64_t rows, int world, int rank, int64_t& b0, int64_t& nb) {
    const int64_t bands = (rows + kBand - 1) / kBand;
    b0 = bands * rank / world;
    nb = bands * (rank + 1) / world - b0;
}

// one source's column tile of the row stripe's band data -> full-width rows
__global__ void k_shard_repack(const uint32_t* __restrict__ rm, const uint16_t* __restrict__ ra,
                               const uint16_t* __restrict__ rb, int nbq, int Wsrc, int Wpsrc, int col0,
                               uint32_t* __restrict__ fm, uint16_t* __restrict__ fa, uint16_t* __restrict__ fb,
                               int Wp) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (c >= Wsrc || b >= nbq) return;
    const int64_t s = (int64_t)b * Wpsrc + c, d = (int64_t)b * Wp + col0 + c;
    fm[d] = rm[s];
    fa[d] = ra[s];
    fb[d] = rb[s];
}

__global__ void k_sum_counts(const unsigned long long* __restrict__ parts, int n, int stride,
                             unsigned long long* __restrict__ total) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long t = 0;
        for (int i = 0; i < n; ++i) t += parts[(int64_t)i * stride];
        *total = t;
    }
}

struct ShardWork {
    const dfc_shard* sh = nullptr;
    int64_t c0, Wg, Wpg;            // column stripe
    int64_t b0, nbq, r0, Hq;        // row stripe
    char* mem = nullptr;
    // column pass products [nb][Wpg]
    uint16_t *first, *last;
    uint32_t* bmask;
    unsigned long long* count;
    // receive area: per source s: masks [nbq][Wp_s] u32, above, below [nbq][Wp_s] u16, count
    std::vector<size_t> roff;
    unsigned long long* rcount;     // [world] (stride 1)
    // full-width band rows of the row stripe
    uint32_t* fm;
    uint16_t *fa, *fb;
    unsigned long long* gcount;
    // band path scratch
    uint32_t *cand, *ent;
    uint16_t* entr;
    int* nent;
    int* cbound;
    cudaEvent_t colpass_done = nullptr, copies_done = nullptr;
};

int64_t rup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

extern "C" {

int dfc_shard_cols(int64_t cols, int world, int rank, int64_t* col0, int64_t* ncols) {
    if (cols < 1 || world < 1 || rank < 0 || rank >= world || !col0 || !ncols) return DFC_ERR_ARG;
    stripe_cols(cols, world, rank, *col0, *ncols);
    return DFC_OK;
}

int dfc_shard_rows(int64_t rows, int world, int rank, int64_t* row0, int64_t* nrows) {
    if (rows < 1 || world < 1 || rank < 0 || rank >= world || !row0 || !nrows) return DFC_ERR_ARG;
    int64_t b0, nb;
    stripe_bands(rows, world, rank, b0, nb);
    *row0 = std::min<int64_t>(rows, b0 * kBand);
    *nrows = std::min<int64_t>(rows, (b0 + nb) * kBand) - *row0;
    return DFC_OK;
}

int dfc_comm_unique_id(uint8_t* id) {
    if (!id) return DFC_ERR_ARG;
    if (!nccl().ok) return DFC_ERR_NCCL;
    ncclUniqueId u;
    const ncclResult_t r = nccl().GetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r);
    memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return DFC_OK;
}

int dfc_comm_init_rank(void** comm, int world, int rank, const uint8_t* id) {
    if (!comm || !id || world < 1 || rank < 0 || rank >= world) return DFC_ERR_ARG;
    if (!nccl().ok) return DFC_ERR_NCCL;
    ncclUniqueId u;
    memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    const ncclResult_t r = nccl().CommInitRank(&c, world, u, rank);
    if (r != ncclSuccess) return nccl_fail(r);
    *comm = c;
    return DFC_OK;
}

int dfc_comm_init_all(void** comms, int ndev, const int* devices) {
    if (!comms || ndev < 1) return DFC_ERR_ARG;
    if (!nccl().ok) return DFC_ERR_NCCL;
    std::vector<ncclComm_t> c((size_t)ndev);
    const ncclResult_t r = nccl().CommInitAll(c.data(), ndev, devices);
    if (r != ncclSuccess) return nccl_fail(r);
    for (int i = 0; i < ndev; ++i) comms[i] = c[(size_t)i];
    return DFC_OK;
}

int dfc_comm_destroy(void* comm) {
    if (!comm) return DFC_OK;
    if (!nccl().ok) return DFC_ERR_NCCL;
    const ncclResult_t r = nccl().CommDestroy(static_cast<ncclComm_t>(comm));
    return r == ncclSuccess ? DFC_OK : nccl_fail(r);
}

int dfc_last_nccl_error(void) { return g_last_nccl; }

int dfc_edt_u8_sharded(const dfc_shard* shards, int n_local, int world, int64_t rows, int64_t cols, int polarity) {
    if (!shards || world < 1 || n_local < 1 || n_local > world) return DFC_ERR_ARG;
    if (polarity != DFC_BG_TO_OBJ && polarity != DFC_OBJ_TO_BG) return DFC_ERR_ARG;
    if (!shape_ok(rows, cols)) return DFC_ERR_SHAPE;
    bool any_comm = false, all_comm = true;
    std::vector<char> seen((size_t)world, 0);
    for (int s = 0; s < n_local; ++s) {
        const dfc_shard& h = shards[s];
        if (h.rank < 0 || h.rank >= world || seen[(size_t)h.rank]) return DFC_ERR_ARG;
        seen[(size_t)h.rank] = 1;
        int64_t c0, w;
        stripe_cols(cols, world, h.rank, c0, w);
        int64_t r0, nr;
        dfc_shard_rows(rows, world, h.rank, &r0, &nr);
        if (w < 1 || !h.d_img || h.pitch_bytes < w || (nr > 0 && !h.d_sqdist)) return DFC_ERR_ARG;
        any_comm |= h.comm != nullptr;
        all_comm &= h.comm != nullptr;
    }
    if (any_comm != all_comm) return DFC_ERR_ARG;
    const bool use_nccl = all_comm;
    if (!use_nccl && n_local != world) return DFC_ERR_ARG;  // in-process exchange: every shard here
    if (use_nccl && !nccl().ok) return DFC_ERR_NCCL;
    int dev0 = 0;
    cudaGetDevice(&dev0);
    g_launches = 0;
    const int64_t H = rows, W = cols, nb = (H + kBand - 1) / kBand, Wp = rup(W, 8);
    const int64_t Ws = rup(W, 32), Ww = (W + 31) / 32;
    std::vector<ShardWork> work((size_t)n_local);
    int rc = DFC_OK;
    bool released = false;
    // scratch release (stream-ordered; in-process copies read the sources, so
    // each stream first waits for every destination's copies)
    auto release = [&]() {
        if (released) return;
        released = true;
        for (ShardWork& w : work) {
            if (!w.sh || !w.mem) continue;
            cudaSetDevice(w.sh->device);
            cudaStream_t st = (cudaStream_t)w.sh->stream;
            for (ShardWork& d : work)
                if (d.copies_done) cudaStreamWaitEvent(st, d.copies_done, 0);
            cudaFreeAsync(w.mem, st);
        }
        for (ShardWork& w : work) {
            if (w.colpass_done) cudaEventDestroy(w.colpass_done);
            if (w.copies_done) cudaEventDestroy(w.copies_done);
        }
        cudaSetDevice(dev0);
    };
    struct Guard {
        std::function<void()> f;
        ~Guard() { f(); }
    } guard{release};
    auto fail = [&](cudaError_t e) {
        rc = cuda_fail(e);
        return rc;
    };

    // ---- 1. allocation + column pass on every local stripe ----
    for (int s = 0; s < n_local && rc == DFC_OK; ++s) {
        ShardWork& w = work[(size_t)s];
        w.sh = &shards[s];
        const dfc_shard& h = *w.sh;
        cudaSetDevice(h.device);
        init_pool_once();
        cudaStream_t st = (cudaStream_t)h.stream;
        stripe_cols(W, world, h.rank, w.c0, w.Wg);
        w.Wpg = rup(w.Wg, 8);
        stripe_bands(H, world, h.rank, w.b0, w.nbq);
        dfc_shard_rows(H, world, h.rank, &w.r0, &w.Hq);
        // layout
        size_t off = 0;
        auto take = [&](size_t bytes) {
            const size_t o = off;
            off += (bytes + 255) & ~(size_t)255;
            return o;
        };
        const size_t o_first = take((size_t)(nb * w.Wpg) * 2), o_last = take((size_t)(nb * w.Wpg) * 2);
        const size_t o_bm = take((size_t)(nb * w.Wpg) * 4), o_cnt = take(8);
        w.roff.assign((size_t)world, 0);
        for (int q = 0; q < world; ++q) {
            int64_t qc0, qw;
            stripe_cols(W, world, q, qc0, qw);
            w.roff[(size_t)q] = take((size_t)(w.nbq * rup(qw, 8)) * 8);
        }
        const size_t o_rcnt = take((size_t)world * 8);
        const size_t o_fm = take((size_t)(w.nbq * Wp) * 4), o_fa = take((size_t)(w.nbq * Wp) * 2),
                     o_fb = take((size_t)(w.nbq * Wp) * 2), o_gc = take(8);
        const int64_t ngroups = (w.nbq + band_group() - 1) / band_group();
        const size_t o_cand = take((size_t)(ngroups * 2 * Ww) * 4), o_ent = take((size_t)(w.Hq * Ws) * 4),
                     o_entr = take((size_t)(w.Hq * Ws) * 2), o_nent = take((size_t)w.Hq * kBandWarps * 4),
                     o_cb = take((size_t)(w.nbq * (kBandWarps + 1)) * 4);
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&w.mem), off, st);
        if (e != cudaSuccess) return fail(e);
        w.first = reinterpret_cast<uint16_t*>(w.mem + o_first);
        w.last = reinterpret_cast<uint16_t*>(w.mem + o_last);
        w.bmask = reinterpret_cast<uint32_t*>(w.mem + o_bm);
        w.count = reinterpret_cast<unsigned long long*>(w.mem + o_cnt);
        w.rcount = reinterpret_cast<unsigned long long*>(w.mem + o_rcnt);
        w.fm = reinterpret_cast<uint32_t*>(w.mem + o_fm);
        w.fa = reinterpret_cast<uint16_t*>(w.mem + o_fa);
        w.fb = reinterpret_cast<uint16_t*>(w.mem + o_fb);
        w.gcount = reinterpret_cast<unsigned long long*>(w.mem + o_gc);
        w.cand = reinterpret_cast<uint32_t*>(w.mem + o_cand);
        w.ent = reinterpret_cast<uint32_t*>(w.mem + o_ent);
        w.entr = reinterpret_cast<uint16_t*>(w.mem + o_entr);
        w.nent = reinterpret_cast<int*>(w.mem + o_nent);
        w.cbound = reinterpret_cast<int*>(w.mem + o_cb);
        const int gl0 = g_launches;
        const int r = column_pass(h.d_img, 1, H, w.Wg, h.pitch_bytes, 0, polarity, 1, nullptr, w.first, w.last,
                                  (int)w.Wpg, st, nullptr, w.count, nullptr, w.bmask, false, true);
        g_launches = gl0 + 2;
        if (r != DFC_OK) return rc = r;
        if (!use_nccl) {
            e = cudaEventCreateWithFlags(&w.colpass_done, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w.copies_done, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventRecord(w.colpass_done, st);
            if (e != cudaSuccess) return fail(e);
        }
    }

    // source s's slices for destination rank q: bands [b0_q, b0_q + nbq_q)
    auto slices = [&](const ShardWork& src, int q, const uint32_t*& m, const uint16_t*& a, const uint16_t*& b,
                      int64_t& n) {
        int64_t qb0, qnb;
        stripe_bands(H, world, q, qb0, qnb);
        m = src.bmask + qb0 * src.Wpg;
        a = src.last + qb0 * src.Wpg;   // nearest object row above the band
        b = src.first + qb0 * src.Wpg;  // ... below
        n = qnb * src.Wpg;
    };
    auto recv_ptrs = [&](const ShardWork& dst, int srank, uint32_t*& m, uint16_t*& a, uint16_t*& b) {
        int64_t sc0, sw;
        stripe_cols(W, world, srank, sc0, sw);
        const int64_t n = dst.nbq * rup(sw, 8);
        char* base = dst.mem + dst.roff[(size_t)srank];
        m = reinterpret_cast<uint32_t*>(base);
        a = reinterpret_cast<uint16_t*>(base + n * 4);
        b = reinterpret_cast<uint16_t*>(base + n * 6);
    };

    // ---- 2. the all-to-all of the band data ----
    if (use_nccl) {
        const NcclApi& nc = nccl();
        ncclResult_t r = nc.GroupStart();
        if (r != ncclSuccess) return nccl_fail(r);
        for (int s = 0; s < n_local; ++s) {
            const ShardWork& w = work[(size_t)s];
            const dfc_shard& h = *w.sh;
            ncclComm_t comm = static_cast<ncclComm_t>(h.comm);
            cudaStream_t st = (cudaStream_t)h.stream;
            for (int q = 0; q < world; ++q) {
                const uint32_t* m;
                const uint16_t *a, *b;
                int64_t n;
                slices(w, q, m, a, b, n);
                uint32_t* rm;
                uint16_t *ra, *rb;
                recv_ptrs(w, q, rm, ra, rb);
                int64_t qc0, qw;
                stripe_cols(W, world, q, qc0, qw);
                const size_t rn = (size_t)(w.nbq * rup(qw, 8));
                // raw bytes (NCCL has no 16-bit integer type)
                if (n > 0) {
                    if ((r = nc.Send(m, (size_t)n * 4, ncclUint8, q, comm, st)) != ncclSuccess) break;
                    if ((r = nc.Send(a, (size_t)n * 2, ncclUint8, q, comm, st)) != ncclSuccess) break;
                    if ((r = nc.Send(b, (size_t)n * 2, ncclUint8, q, comm, st)) != ncclSuccess) break;
                }
                if ((r = nc.Send(w.count, 8, ncclUint8, q, comm, st)) != ncclSuccess) break;
                if (rn > 0) {
                    if ((r = nc.Recv(rm, rn * 4, ncclUint8, q, comm, st)) != ncclSuccess) break;
                    if ((r = nc.Recv(ra, rn * 2, ncclUint8, q, comm, st)) != ncclSuccess) break;
                    if ((r = nc.Recv(rb, rn * 2, ncclUint8, q, comm, st)) != ncclSuccess) break;
                }
                if ((r = nc.Recv(w.rcount + q, 8, ncclUint8, q, comm, st)) != ncclSuccess) break;
            }
            if (r != ncclSuccess) break;
        }
        const ncclResult_t r2 = nc.GroupEnd();
        if (r != ncclSuccess) return nccl_fail(r);
        if (r2 != ncclSuccess) return nccl_fail(r2);
    } else {
        for (int d = 0; d < n_local; ++d) {
            const ShardWork& dst = work[(size_t)d];
            cudaStream_t st = (cudaStream_t)dst.sh->stream;
            cudaSetDevice(dst.sh->device);
            for (int s = 0; s < n_local; ++s) {
                const ShardWork& src = work[(size_t)s];
                cudaError_t e = cudaStreamWaitEvent(st, src.colpass_done, 0);
                const uint32_t* m;
                const uint16_t *a, *b;
                int64_t n;
                slices(src, dst.sh->rank, m, a, b, n);
                uint32_t* rm;
                uint16_t *ra, *rb;
                recv_ptrs(dst, src.sh->rank, rm, ra, rb);
                const int dd = dst.sh->device, sd = src.sh->device;
                if (e == cudaSuccess && n > 0) e = cudaMemcpyPeerAsync(rm, dd, m, sd, (size_t)n * 4, st);
                if (e == cudaSuccess && n > 0) e = cudaMemcpyPeerAsync(ra, dd, a, sd, (size_t)n * 2, st);
                if (e == cudaSuccess && n > 0) e = cudaMemcpyPeerAsync(rb, dd, b, sd, (size_t)n * 2, st);
                if (e == cudaSuccess) e = cudaMemcpyPeerAsync(dst.rcount + src.sh->rank, dd, src.count, sd, 8, st);
                if (e != cudaSuccess) return fail(e);
            }
            cudaError_t e = cudaEventRecord(dst.copies_done, st);
            if (e != cudaSuccess) return fail(e);
        }
    }

    // ---- 3. repack + band path on every local row stripe ----
    for (int s = 0; s < n_local; ++s) {
        ShardWork& w = work[(size_t)s];
        const dfc_shard& h = *w.sh;
        cudaSetDevice(h.device);
        cudaStream_t st = (cudaStream_t)h.stream;
        k_sum_counts<<<1, 32, 0, st>>>(w.rcount, world, 1, w.gcount);
        ++g_launches;
        if (w.Hq > 0) {
            for (int q = 0; q < world; ++q) {
                uint32_t* rm;
                uint16_t *ra, *rb;
                recv_ptrs(w, q, rm, ra, rb);
                int64_t qc0, qw;
                stripe_cols(W, world, q, qc0, qw);
                const dim3 grid((unsigned)((qw + 255) / 256), (unsigned)w.nbq);
                k_shard_repack<<<grid, 256, 0, st>>>(rm, ra, rb, (int)w.nbq, (int)qw, (int)rup(qw, 8), (int)qc0, w.fm,
                                                     w.fa, w.fb, (int)Wp);
                ++g_launches;
            }
            RowArgs a{};
            a.W = (int)W;
            a.H = (int)w.Hq;
            a.total_rows = w.Hq;
            a.D = reinterpret_cast<char*>(h.d_sqdist);
            a.S = reinterpret_cast<char*>(h.d_dist);
            a.LB = reinterpret_cast<char*>(h.d_label);
            a.vec = W % 4 == 0 && (uintptr_t)h.d_sqdist % 16 == 0 && (!h.d_dist || (uintptr_t)h.d_dist % 16 == 0) &&
                    (!h.d_label || (uintptr_t)h.d_label % 16 == 0);
            BandArgs ba;
            ba.bmask = w.fm;
            ba.above = w.fa;
            ba.below = w.fb;
            ba.cand = w.cand;
            ba.counts = w.gcount;
            ba.ent = w.ent;
            ba.entr = w.entr;
            ba.nent = w.nent;
            ba.cbound = w.cbound;
            ba.Ws = Ws;
            ba.H = (int)w.Hq;
            ba.W = (int)W;
            ba.Wp = (int)Wp;
            ba.nb = (int)w.nbq;
            ba.Ww = (int)Ww;
            ba.n_img = 1;
            ba.pol0 = polarity;
            ba.nplanes = 1;
            ba.band0 = (int)w.b0;
            ba.Hg = (int)H;
            ba.group = band_group();
            ba.ngroups = (int)((w.nbq + ba.group - 1) / ba.group);
            ba.pts_gate = false;
            ba.all_planes = true;
            const int r = launch_band_path(a, ba, false, st);
            if (r != DFC_OK) return rc = r;
        }
    }

    release();
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? rc : cuda_fail(e);
}

}  // extern "C"
