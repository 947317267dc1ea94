// dfc_api.cu -- the extern "C" entry points declared in include/distfield_cuda.h.
//
// Plumbing only: argument validation, scratch from the stream-ordered memory
// pool, launch geometry, status codes.  Never throws, never synchronises.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "dfc_kernels.cuh"



using namespace dfc;

namespace {

thread_local int g_last_cuda = 0;
thread_local int g_launches = 0;
thread_local cudaEvent_t g_ev[3] = {nullptr, nullptr, nullptr};
thread_local int g_lr_chunk = 0;  // k_rows_lr columns per warp chunk (0: default)
thread_local int64_t g_band_min_px = -1;  // smallest image the band path takes (-1: default)
thread_local int g_row_mode = 0;  // 0: default, 1: segment/merge kernel, 4: dense rows first, the
                                  // rest by the segment kernel, 5: lane-per-row, 6: anchored (default)

// DFC_ROWS=segment|stream overrides the default stage-2 kernel (tuning/A-B).
int env_row_mode() {
    static const int m = [] {
        const char* v = getenv("DFC_ROWS");
        if (v && strcmp(v, "segment") == 0) return 1;
        if (v && strcmp(v, "dense") == 0) return 4;
        if (v && strcmp(v, "lr") == 0) return 5;
        if (v && strcmp(v, "anc") == 0) return 6;
        // default: point planes, dense rows, sparse planes, then anchored
        // segments for the rest (k_rows where those do not apply)
        return 6;
    }();
    return m;
}

void prof(int k, cudaStream_t st) {
    if (g_ev[k]) cudaEventRecord(g_ev[k], st);
}

constexpr int kMaxRowCols = 32768;  // widest row the shared-memory row pass holds

int cuda_fail(cudaError_t e) {
    g_last_cuda = (int)e;
    return DFC_ERR_CUDA;
}

bool shape_ok(int64_t rows, int64_t cols) {
    if (rows < 1 || cols < 1 || rows > 65535 || cols > kMaxRowCols) return false;
    const int64_t b = (rows - 1) * (rows - 1) + (cols - 1) * (cols - 1);
    return b <= DFC_MAX_SQDIST;
}

bool aligned(const void* p, int a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Keep freed scratch in the pool: after the first call on a device no
// cudaMalloc happens.  Once per device, thread-safe (a single process may
// drive several GPUs, dfc_edt_u8_sharded).
void init_pool_once() {
    constexpr int kMaxDev = 64;
    static std::once_flag flags[kMaxDev];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return;
    std::call_once(flags[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        if (const char* v = getenv("DFC_SPARSE_DIV")) {  // tuning: the sparse-plane gate
            const unsigned long long d = strtoull(v, nullptr, 10);
            if (d >= 1) cudaMemcpyToSymbol(dfc::c_sparse_div, &d, sizeof(d));
        }
    });
}

// DFC_DEBUG_GUARD=1 (debug; compute-sanitizer's stand-in where that tool is
// unavailable): every scratch allocation gets a kGuard-byte canary zone on
// both sides and a poisoned interior (0xCD: a kernel that reads scratch it
// never wrote computes garbage and fails parity); when the allocation is
// released a kernel counts the canary bytes that changed.  The count is read
// with dfc_debug_guard_violations().
constexpr size_t kGuard = 65536;
__device__ unsigned long long g_guard_bad;

bool guard_on() {
    static const bool on = [] {
        const char* v = getenv("DFC_DEBUG_GUARD");
        return v && v[0] == '1';
    }();
    return on;
}

__global__ void k_guard_check(const uint8_t* lo, const uint8_t* hi, size_t n) {
    unsigned bad = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        bad += (lo[i] != 0xA5) + (hi[i] != 0xA5);
    if (bad) atomicAdd(&g_guard_bad, (unsigned long long)bad);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize, raised once per (device,
// kernel) instead of on every call (the attribute is per context; a call only
// needs it to be at least its own request).
cudaError_t set_dyn_smem(const void* fn, int bytes) {
    constexpr int kMaxDev = 64;
    static std::mutex mu;
    static std::unordered_map<const void*, int> cur[kMaxDev];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev)
        return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    std::lock_guard<std::mutex> lock(mu);
    int& have = cur[dev][fn];
    if (bytes <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

struct Scratch {
    void* p = nullptr;
    void* raw = nullptr;
    size_t bytes = 0;
    cudaStream_t st;
    explicit Scratch(cudaStream_t s) : st(s) {}
    cudaError_t alloc(size_t n) {
        if (!guard_on()) return cudaMallocAsync(&p, n, st);
        bytes = (n + 255) / 256 * 256;
        cudaError_t e = cudaMallocAsync(&raw, bytes + 2 * kGuard, st);
        if (e != cudaSuccess) return e;
        char* c = static_cast<char*>(raw);
        p = c + kGuard;
        if ((e = cudaMemsetAsync(c, 0xA5, kGuard, st)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(c + kGuard, 0xCD, bytes, st)) != cudaSuccess) return e;
        return cudaMemsetAsync(c + kGuard + bytes, 0xA5, kGuard, st);
    }
    ~Scratch() {
        if (raw) {
            const uint8_t* c = static_cast<const uint8_t*>(raw);
            k_guard_check<<<64, 256, 0, st>>>(c, c + kGuard + bytes, kGuard);
            cudaFreeAsync(raw, st);
        } else if (p) {
            cudaFreeAsync(p, st);
        }
    }
};

struct RowGeom {
    int T, L, R, row_words, smem_bytes;
};

// T threads per row (power of two, 32..1024), L = 2^k columns per thread.
// Shared memory holds a whole row (~6 B/column), so the rows resident per SM
// are fixed by W; long segments (L up to 128) keep the merge tree shallow.
// DFC_ROW_L (env) overrides the target segment length for tuning.
RowGeom row_geom(int W) {
    static int target = [] {
        const char* e = getenv("DFC_ROW_L");
        const int v = e ? atoi(e) : 0;
        return (v == 4 || v == 8 || v == 16 || v == 32 || v == 64 || v == 128) ? v : 32;
    }();
    RowGeom g;
    g.T = 32;
    while (g.T < 1024 && (int64_t)g.T * target < W) g.T <<= 1;
    const int per = (W + g.T - 1) / g.T;
    g.L = 4;
    while (g.L < per) g.L <<= 1;
    static int cta = [] {  // threads per CTA target (DFC_ROW_CTA, tuning)
        const char* e = getenv("DFC_ROW_CTA");
        const int v = e ? atoi(e) : 0;
        return (v == 32 || v == 64 || v == 128 || v == 256 || v == 512) ? v : 64;
    }();
    g.R = g.T >= cta ? 1 : cta / g.T;
    g.row_words = dfc::row_words(g.T, g.L);
    g.smem_bytes = g.R * g.row_words * 4;
    // keep the CTA within the 227 KB opt-in limit: fewer rows per CTA
    while (g.R > 1 && g.smem_bytes > 227 * 1024) {
        g.R >>= 1;
        g.smem_bytes = g.R * g.row_words * 4;
    }
    return g;
}

// Stage 1 into a uint16 nearest-row plane [npol][n][H][Wp].
int column_pass(const uint8_t* img, int64_t n, int64_t H, int64_t W, int64_t pitch, int64_t istride,
                int pol0, int npol, uint16_t* nr, uint16_t* first, uint16_t* last, int Wp,
                cudaStream_t st, int32_t* vsq = nullptr, unsigned long long* counts = nullptr,
                uint32_t* pts = nullptr, uint32_t* bmask = nullptr, bool skip_full = false,
                bool no_fill = false, bool skip_sparse = false, uint32_t* objcol = nullptr) {
    ColArgs c;
    c.img = img;
    c.pitch = pitch;
    c.img_stride = istride;
    c.n_img = (int)n;
    c.H = (int)H;
    c.W = (int)W;
    c.Wp = Wp;
    c.nb = (int)((H + kBand - 1) / kBand);
    c.pol0 = pol0;
    c.npol = npol;
    c.vec = aligned(img, 4) && pitch % 4 == 0 && istride % 4 == 0;
    c.pts = counts ? pts : nullptr;
    c.pcounts = counts;
    c.bmask = bmask;
    c.skip_full = skip_full && bmask != nullptr && counts != nullptr;
    c.skip_sparse = skip_sparse && bmask != nullptr && counts != nullptr;
    c.objcol = objcol;
    const unsigned long long* skip = c.pts ? counts : nullptr;
    const int tpb = 128;
    dim3 grid((unsigned)(((W + 3) / 4 + tpb - 1) / tpb), (unsigned)c.nb, (unsigned)n);
    if (counts) {
        const cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)npol * n * sizeof(unsigned long long), st);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    k_band_summary<<<grid, tpb, 0, st>>>(c, first, last, counts);
    if (c.nb <= 64) {  // short columns: serial over bands, one thread per column
        dim3 gs((unsigned)((W + 255) / 256), (unsigned)(npol * n));
        k_band_scan_serial<<<gs, 256, 0, st>>>((int)W, Wp, c.nb, npol * n, first, last, skip);
    } else {           // tall columns: chunks of bands scanned in parallel
        const int nc = std::min(32, c.nb / 4);
        dim3 gs((unsigned)((W + 127) / 128), (unsigned)(npol * n));
        k_band_scan<<<gs, 32 * nc, 0, st>>>((int)W, Wp, c.nb, npol * n, first, last, skip);
    }
    if (no_fill) {  // the row pass stages from the bands: no nearest-row plane
        g_launches += 2;
        return DFC_OK;
    }
    // several bands per CTA for batches (a skipped plane costs few CTAs); for a
    // single image ~8 CTAs per SM in all (each CTA walks nb / grid.y bands), so
    // a plane the row pass reads from the bands costs ~1k early exits, not
    // one per (band, 512 columns)
    const unsigned fy = n > 1 ? (unsigned)((c.nb + kFillBands - 1) / kFillBands)
                              : (unsigned)std::max<int64_t>(1, std::min<int64_t>(c.nb, (148 * 8 + grid.x - 1) / grid.x));
    const dim3 fgrid(grid.x, fy, grid.z);
    if (vsq)
        k_band_fill<true><<<fgrid, tpb, 0, st>>>(c, first, last, nullptr, vsq);
    else
        k_band_fill<false><<<fgrid, tpb, 0, st>>>(c, first, last, nr, nullptr);
    g_launches += 3;
    return DFC_OK;
}

struct OutSet {
    int32_t* D[2] = {nullptr, nullptr};
    float* S[2] = {nullptr, nullptr};
    int32_t* LB[2] = {nullptr, nullptr};
    int32_t* NC[2] = {nullptr, nullptr};
};

bool out_vec_ok(const void* p, int64_t stride) {
    return p == nullptr || (aligned(p, 16) && stride % 16 == 0);
}

// dense planes by k_rows_anc too (all-object segments and anchors on object
// pixels are free there); DFC_ANC_DENSE=0 keeps k_rows_dense (A/B)
bool anc_dense_on() {
    static const bool on = [] {
        const char* v = getenv("DFC_ANC_DENSE");
        return !(v && v[0] == '0');
    }();
    return on;
}

// Band source of k_rows_anc (see RowArgs): masks [img][nb][Wp], carries
// above / below [plane][nb][Wp] of this call's planes, first polarity.
struct BandSrc {
    const uint32_t* bmask = nullptr;   // K1a's masks (single images), else null
    const uint16_t* above = nullptr;
    const uint16_t* below = nullptr;
    uint32_t* objcol = nullptr;        // K1a's object-column bits of these planes (band path), else null
    int nb = 0, n_img = 1, pol0 = 0;
    bool anc = false;     // k_rows_anc stages its rows from the bands
    bool sparse = false;  // the band path (k_rows_band.cu) takes the sparse planes
};

// Bands per candidate group of the band path (k_hull<2>): DFC_BAND_GROUP
// (tuning), default 4.
int band_group() {
    static const int g = [] {
        const char* v = getenv("DFC_BAND_GROUP");
        const int x = v ? atoi(v) : 0;
        return x >= 1 && x <= 64 ? x : 4;
    }();
    return g;
}

// The band path (six launches, ~60 us of latency-bound stages even when every
// CTA exits at once) is only offered images above this size: DFC_BAND_MIN_PX
// (tuning) or dfc_set_band_min_pixels, default 2^24 + 1 -- larger than 4096^2.
// Smaller sparse planes keep the lane-per-row kernel (k_rows_lr).
int64_t band_min_px() {
    static const int64_t env = [] {
        const char* v = getenv("DFC_BAND_MIN_PX");
        return v ? (int64_t)strtoll(v, nullptr, 10) : (int64_t)-1;
    }();
    if (g_band_min_px >= 0) return g_band_min_px;
    return env >= 0 ? env : ((int64_t)1 << 24) + 1;
}

// DFC_SPARSE=lr keeps the lane-per-row chunk scan (k_rows_lr, from the
// nearest-row plane) for sparse planes instead of the band path (A/B)
bool band_sparse_on() {
    static const bool on = [] {
        const char* v = getenv("DFC_SPARSE");
        return !(v && strcmp(v, "lr") == 0);
    }();
    return on;
}

// Per-device helper stream of the default row pass: when the band path is on,
// the kernel families of the planes it does NOT take (point planes, the rows of
// non-sparse planes) are enqueued on it, beside the band path on the caller's
// stream -- for a sparse image those launches find no plane of theirs, and
// their launch latencies no longer sit in front of the band path (C5: ~25 us).
// Fork / join by events only: no host synchronisation, legal under stream
// capture.  The mutex serialises the host-side enqueue per device (the events
// are shared).  DFC_AUX_STREAM=0 keeps everything on the caller's stream.
struct AuxPipe {
    std::mutex mu;
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    bool ok = false;
};
AuxPipe* aux_pipe() {
    static const bool on = [] {
        const char* v = getenv("DFC_AUX_STREAM");
        return !(v && v[0] == '0');
    }();
    if (!on) return nullptr;
    constexpr int kMaxDev = 64;
    static AuxPipe pipes[kMaxDev];
    static std::once_flag flags[kMaxDev];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
    AuxPipe* ap = &pipes[dev];
    std::call_once(flags[dev], [ap] {
        bool ok = cudaStreamCreateWithFlags(&ap->aux, cudaStreamNonBlocking) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&ap->fork, cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&ap->join, cudaEventDisableTiming) == cudaSuccess;
        ap->ok = ok;
        if (!ok) cudaGetLastError();
    });
    return ap->ok ? ap : nullptr;
}
// fork at construction, join (the caller's stream waits for the helper) at scope exit
struct AuxScope {
    AuxPipe* ap;
    cudaStream_t st;
    std::unique_lock<std::mutex> lock;
    AuxScope(AuxPipe* p, cudaStream_t s) : ap(p), st(s) {
        if (!ap) return;
        lock = std::unique_lock<std::mutex>(ap->mu);
        if (cudaEventRecord(ap->fork, st) != cudaSuccess || cudaStreamWaitEvent(ap->aux, ap->fork, 0) != cudaSuccess) {
            cudaGetLastError();
            lock.unlock();
            ap = nullptr;
        }
    }
    cudaStream_t stream() const { return ap ? ap->aux : st; }
    ~AuxScope() {
        if (!ap) return;
        cudaEventRecord(ap->join, ap->aux);
        cudaStreamWaitEvent(st, ap->join, 0);
    }
};

template <bool TN, int DO>
cudaError_t launch_rows_fill(const RowArgs& a, const BandArgs& ba, unsigned grid, int smem, cudaStream_t st) {
    cudaError_t e = set_dyn_smem((const void*)(k_band_rows_fill<TN, DO>), smem);
    if (e != cudaSuccess) return e;
    k_band_rows_fill<TN, DO><<<grid, 32 * kBandWarps, smem, st>>>(a, ba);
    return cudaSuccess;
}

// The band path (k_rows_band.cu) over the sparse planes of `ba`: object-column
// runs, hull filter (coarse lines, then the groups' lines), per-row stacks and
// fill into a's outputs.
int launch_band_path(const RowArgs& a, const BandArgs& ba_in, bool take_new, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    BandArgs ba = ba_in;
    ba.cbands = ba.group >= kCoarseBands ? ba.group : kCoarseBands / ba.group * ba.group;
    ba.ncoarse = (ba.nb + ba.cbands - 1) / ba.cbands;
    Scratch hs(st);
    const size_t oc_bytes = (size_t)round_up((int64_t)ba.nplanes * ba.nb * ba.Ww * 4, 256);
    const size_t co_bytes = (size_t)round_up((int64_t)ba.nplanes * ba.ncoarse * 2 * ba.Ww * 4, 256);
    const bool have_oc = ba_in.objcol != nullptr;  // K1a wrote the object-column bits
    e = hs.alloc((have_oc ? 2 : 3) * oc_bytes + co_bytes);
    if (e != cudaSuccess) return cuda_fail(e);
    ba.objpre = static_cast<uint32_t*>(hs.p);
    ba.objsuf = reinterpret_cast<uint32_t*>(static_cast<char*>(hs.p) + oc_bytes);
    ba.coarse = reinterpret_cast<uint32_t*>(static_cast<char*>(hs.p) + 2 * oc_bytes);
    if (!have_oc) {
        ba.objcol = reinterpret_cast<uint32_t*>(static_cast<char*>(hs.p) + 2 * oc_bytes + co_bytes);
        k_band_objcols<<<dim3((unsigned)((ba.Ww * 32 + 255) / 256), (unsigned)std::min(ba.nb, 64), (unsigned)ba.nplanes), 256, 0, st>>>(ba);
        ++g_launches;
    }
    const int nwin = (ba.Ww + 31) / 32;
    k_objcol_runs<<<dim3((unsigned)((ba.Ww + 127) / 128), (unsigned)ba.ncoarse, (unsigned)ba.nplanes), 128, 0, st>>>(ba);
    k_hull<0><<<(unsigned)((int64_t)ba.nplanes * ba.ncoarse * 2 * nwin), kHullThreads, 0, st>>>(ba);
    k_hull<1><<<(unsigned)((int64_t)ba.nplanes * ba.ncoarse * 2), kHullThreads, 0, st>>>(ba);
    k_hull<2><<<(unsigned)((int64_t)ba.nplanes * ba.ngroups * 2), kHullThreads, 0, st>>>(ba);
    g_launches += 4;

    const int donly = a.D && !a.LB && !a.NC ? (a.S ? 2 : 1) : 0;  // values only (D, optionally sqrt D)
    const int64_t tasks = (int64_t)ba.nplanes * ba.nb;
    {
        const unsigned g = (unsigned)tasks;
        // CTAs per SM of the fused kernel, by shared memory (DFC_BAND_OCC, tuning):
        // measured on C5: 4 (the stack phases need the parallelism) 1.356 ms, 3 1.451, 2 1.533, 1 2.082
        static const int occ = [] {
            const char* v = getenv("DFC_BAND_OCC");
            const int x = v ? atoi(v) : 0;
            return x >= 1 && x <= 4 ? x : 4;
        }();
        const int rsm = std::max(band_fused_smem_bytes(), std::min(227 * 1024, (228 * 1024) / occ - 1024 - 1024) / 16 * 16);
        if (take_new)
            e = donly == 1 ? launch_rows_fill<true, 1>(a, ba, g, rsm, st)
                           : donly == 2 ? launch_rows_fill<true, 2>(a, ba, g, rsm, st) : launch_rows_fill<true, 0>(a, ba, g, rsm, st);
        else
            e = donly == 1 ? launch_rows_fill<false, 1>(a, ba, g, rsm, st)
                           : donly == 2 ? launch_rows_fill<false, 2>(a, ba, g, rsm, st) : launch_rows_fill<false, 0>(a, ba, g, rsm, st);
        if (e != cudaSuccess) return cuda_fail(e);
        ++g_launches;
    }
    return DFC_OK;
}

// Stage 2 over `nimg` planes of H rows.  Plane b writes its outputs at
// base + b*stride.  take_new selects meijster_scan's tie rule.
int row_pass(const uint16_t* nr, int64_t nimg, int64_t H, int64_t W, int Wp, bool take_new,
             int32_t* D, int64_t sD, float* S, int64_t sS, int32_t* LB, int64_t sL, int32_t* NC,
             int64_t sN, cudaStream_t st, bool vdist = false, int tile_cols = 0,
             int64_t tile_stride = 0, int row0 = 0, const unsigned long long* plane_counts = nullptr,
             const uint32_t* pts = nullptr, const BandSrc& band = BandSrc()) {
    const RowGeom g = row_geom((int)W);
    RowArgs a;
    a.nr = nr;
    a.nr_img_stride = H * Wp;
    a.Wp = Wp;
    a.tile_cols = tile_cols > 0 ? tile_cols : Wp;
    a.tile_stride = tile_stride;
    a.row0 = row0;
    a.H = (int)H;
    a.W = (int)W;
    a.total_rows = nimg * H;
    a.T = g.T;
    a.L = g.L;
    a.R = g.R;
    a.row_smem_words = g.row_words;
    a.D = reinterpret_cast<char*>(D);
    a.sD = sD;
    a.S = reinterpret_cast<char*>(S);
    a.sS = sS;
    a.LB = reinterpret_cast<char*>(LB);
    a.sL = sL;
    a.NC = reinterpret_cast<char*>(NC);
    a.sN = sN;
    a.vdist = vdist;
    a.vec = W % 4 == 0 && out_vec_ok(D, sD) && out_vec_ok(S, sS) && out_vec_ok(LB, sL) &&
            out_vec_ok(NC, sN);
    a.row_list = nullptr;
    a.row_count = nullptr;
    a.vec_nr = false;
    a.row_done = nullptr;
    a.lr_gate = false;
    a.pts_gate = false;
    a.plane_counts = plane_counts;
    a.bmask = nullptr;
    a.babove = a.bbelow = nullptr;
    a.nb = band.nb;
    a.n_img = band.n_img;
    a.bpol0 = band.pol0;
    const int mode = g_row_mode != 0 ? g_row_mode : env_row_mode();
    const int64_t blocks = (a.total_rows + g.R - 1) / g.R;
    if (blocks > 0x7fffffff) return DFC_ERR_SHAPE;
    const void* fn = take_new ? rows_kernel_ptr<true>(g.L) : rows_kernel_ptr<false>(g.L);
    cudaError_t e = set_dyn_smem((const void*)(fn), g.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e);

    // Lane-per-row chunk scan (k_rows_lr.cu): needs 16-byte nr loads.
    const bool lr_ok = aligned(nr, 16) && Wp % 8 == 0 && a.tile_cols % 8 == 0 && a.tile_stride % 8 == 0 &&
                       a.nr_img_stride % 8 == 0;
    static const int chunk_env = [] {  // DFC_LR_CHUNK (tuning): columns per warp chunk
        const char* v = getenv("DFC_LR_CHUNK");
        const int c = v ? atoi(v) : 0;
        return c >= 32 ? c & ~31 : 0;
    }();
    // chunk: a multiple of 32 columns.  Default: as wide as ~4096 warps allow
    // (every chunk boundary costs two owner searches), at least 256 columns.
    int lrC = g_lr_chunk > 0 ? g_lr_chunk : chunk_env;
    if (lrC == 0) {
        const int64_t bands = (a.total_rows + 31) / 32;
        const int64_t nch = std::max<int64_t>(1, (4096 + bands - 1) / bands);
        lrC = 256;
        while (lrC < 32768 && (int64_t)lrC * nch < W) lrC <<= 1;
    }
    lrC = (int)std::min<int64_t>(round_up(W, 32), lrC);
    const int lrWs = (int)round_up(W, 32);  // scratch row stride (16-byte granules of both lists)
    const size_t ent_bytes = (size_t)round_up(a.total_rows * lrWs * 4, 256);
    const size_t entr_bytes = (size_t)round_up(a.total_rows * lrWs * 2, 256);
    auto launch_lr = [&](RowArgs la, void* scratch, int* fail_rows, int* fail_count, cudaStream_t ls) -> int {
        const int64_t nchunks = (W + lrC - 1) / lrC;
        const int64_t warps = (la.total_rows + 31) / 32 * nchunks;
        const int64_t lblocks = (warps + kLrWarps - 1) / kLrWarps;
        if (lblocks > 0x7fffffff) return DFC_ERR_SHAPE;
        uint32_t* ent = static_cast<uint32_t*>(scratch);
        uint16_t* entr = reinterpret_cast<uint16_t*>(static_cast<char*>(scratch) + ent_bytes);
        const void* lfn = take_new ? lr_kernel_ptr<true>() : lr_kernel_ptr<false>();
        const int lsm = lr_smem_bytes();
        cudaError_t le = set_dyn_smem((const void*)(lfn), lsm);
        if (le != cudaSuccess) return cuda_fail(le);
        int Cc = lrC, Wsc = lrWs;
        void* largs[] = {&la, &ent, &entr, &Wsc, &Cc, &fail_rows, &fail_count};
        le = cudaLaunchKernel(lfn, dim3((unsigned)lblocks), dim3(32 * kLrWarps), largs, (size_t)lsm, ls);
        if (le != cudaSuccess) return cuda_fail(le);
        ++g_launches;
        return DFC_OK;
    };

    // Mode 5: every row by k_rows_lr; rows whose live stack overflows (flagged
    // 2 in row_done -- once per row, however many of its chunks overflow) are
    // compacted into a list and recomputed by k_rows.
    if (mode == 5 && lr_ok) {
        Scratch fl(st);
        const size_t flag_bytes = (size_t)round_up(a.total_rows, 256);
        e = fl.alloc(ent_bytes + entr_bytes + flag_bytes + (size_t)(a.total_rows + 1) * sizeof(int));
        if (e != cudaSuccess) return cuda_fail(e);
        uint8_t* flags = reinterpret_cast<uint8_t*>(static_cast<char*>(fl.p) + ent_bytes + entr_bytes);
        int* fail_count = reinterpret_cast<int*>(flags + flag_bytes);
        int* fail_rows = fail_count + 1;
        e = cudaMemsetAsync(flags, 0, flag_bytes + sizeof(int), st);
        if (e != cudaSuccess) return cuda_fail(e);
        RowArgs la = a;
        la.lr_gate = false;
        la.row_done = flags;
        int rc = launch_lr(la, fl.p, nullptr, nullptr, st);
        if (rc != DFC_OK) return rc;
        const int64_t rblocks = std::min<int64_t>((a.total_rows + 255) / 256, 148 * 8);
        k_rows_failed<<<(unsigned)rblocks, 256, 0, st>>>(flags, a.total_rows, fail_rows, fail_count);
        ++g_launches;
        RowArgs fb = a;  // fallback: the segment kernel over the overflowed rows
        fb.row_list = fail_rows;
        fb.row_count = fail_count;
        void* fargs[] = {&fb};
        const int64_t fblocks = std::min<int64_t>(blocks, 148 * 4);
        e = cudaLaunchKernel(fn, dim3((unsigned)fblocks), dim3(g.R * g.T), fargs, (size_t)g.smem_bytes, st);
        if (e != cudaSuccess) return cuda_fail(e);
        ++g_launches;
        return DFC_OK;
    }

    // Default (6): per plane by its object count (column pass) -- point planes
    // by k_rows_pts, sparse planes (< 1/256) by k_rows_lr, every other row by
    // k_rows_anc.  Where k_rows_anc does not apply (rows wider than kAncMaxW,
    // column-tiled planes) and in mode 4: dense planes (>= 50% object pixels,
    // W <= kDenseMaxW) by k_rows_dense and the rest by k_rows.
    if (mode == 4 || mode == 6) {
        // anchored segments (k_rows_anc.cu) for every row the point / sparse
        // kernels do not own: one tile, W <= kAncMaxW
        const bool anc_on = mode == 6 && W <= kAncMaxW && a.tile_cols >= W && row0 == 0 && H <= 32768;
        const bool dense_on = W <= kDenseMaxW && !(anc_on && anc_dense_on());
        // sparse planes: the band path when the column pass left its band masks
        const bool band_on = mode == 6 && band.sparse && band.bmask && plane_counts != nullptr &&
                             a.tile_cols >= W && row0 == 0;
        const bool lr_on = lr_ok && plane_counts != nullptr && !band_on;
        const int64_t Ww = (W + 31) / 32;
        const int bgroup = band_group();
        const int64_t ngroups = (band.nb + bgroup - 1) / bgroup;
        const size_t cand_bytes = band_on ? (size_t)round_up(nimg * ngroups * 2 * Ww * 4, 256) : 0;
        const size_t nent_bytes = band_on ? (size_t)round_up(a.total_rows * kBandWarps * 4, 256) +
                                                (size_t)round_up(nimg * band.nb * (kBandWarps + 1) * 4, 256)
                                          : 0;
        Scratch fl(st);
        const size_t flag_bytes = (size_t)round_up(a.total_rows, 256);
        const size_t list_bytes = (size_t)round_up((a.total_rows + 1) * 4, 256);
        e = fl.alloc(flag_bytes + list_bytes + (lr_on || band_on ? ent_bytes + entr_bytes : 0) + cand_bytes +
                     nent_bytes);
        if (e != cudaSuccess) return cuda_fail(e);
        a.row_done = static_cast<uint8_t*>(fl.p);
        int* rest_count = reinterpret_cast<int*>(static_cast<char*>(fl.p) + flag_bytes);
        int* rest_rows = rest_count + 1;
        e = cudaMemsetAsync(a.row_done, 0, flag_bytes + 4, st);  // flags and the list count
        if (e != cudaSuccess) return cuda_fail(e);
        a.lr_gate = lr_on;
        a.pts_gate = pts != nullptr && plane_counts != nullptr && H % 32 == 0;
        // the families beside the band path go to the helper stream (joined at scope exit,
        // before `fl` is released)
        // (batches of point planes, C3: the point kernel stays on the caller's stream and
        // the families that find no plane of theirs go beside it)
        const bool pts_main = !band_on && a.pts_gate && nimg > 1;
        AuxScope aux(band_on || pts_main ? aux_pipe() : nullptr, st);
        const cudaStream_t os = aux.stream();
        if (a.pts_gate) {  // point planes: from K1a's object list, no nearest-row plane
            const void* pfn = take_new ? pts_kernel_ptr<true>() : pts_kernel_ptr<false>();
            const int64_t pblocks = ((a.total_rows + 31) / 32 + kPtsWarps - 1) / kPtsWarps;
            void* pargs[] = {&a, &pts};
            e = cudaLaunchKernel(pfn, dim3((unsigned)pblocks), dim3(32 * kPtsWarps), pargs, 0, pts_main ? st : os);
            if (e != cudaSuccess) return cuda_fail(e);
            ++g_launches;
        }
        if (dense_on) {  // dense rows (short runs between object pixels): flagged 1
            a.vec_nr = aligned(nr, 16) && Wp % 8 == 0 && a.nr_img_stride % 8 == 0 && a.tile_cols >= W;
            const void* dfn = take_new ? dense_kernel_ptr<true>() : dense_kernel_ptr<false>();
            const int dsm = dense_smem_bytes((int)W);
            e = set_dyn_smem((const void*)(dfn), dsm);
            if (e != cudaSuccess) return cuda_fail(e);
            const int64_t dblocks = std::min<int64_t>((a.total_rows + kDenseWarps - 1) / kDenseWarps, 148 * 16);
            void* dargs[] = {&a};
            e = cudaLaunchKernel(dfn, dim3((unsigned)dblocks), dim3(32 * kDenseWarps), dargs, (size_t)dsm, os);
            if (e != cudaSuccess) return cuda_fail(e);
            ++g_launches;
        }
        if (lr_on) {  // rows of sparse planes; overflowed rows flagged 2
            const int rc = launch_lr(a, static_cast<char*>(fl.p) + flag_bytes + list_bytes, nullptr, nullptr, os);
            if (rc != DFC_OK) return rc;
        }
        a.lr_gate = lr_on || band_on;  // the other kernels skip the sparse planes' rows
        if (band_on) {  // sparse planes: candidates per band, per-row stacks, fill
            char* base = static_cast<char*>(fl.p) + flag_bytes + list_bytes;
            BandArgs ba;
            ba.bmask = band.bmask;
            ba.above = band.above;
            ba.below = band.below;
            ba.objcol = band.objcol;
            ba.ent = reinterpret_cast<uint32_t*>(base);
            ba.entr = reinterpret_cast<uint16_t*>(base + ent_bytes);
            ba.cand = reinterpret_cast<uint32_t*>(base + ent_bytes + entr_bytes);
            ba.nent = reinterpret_cast<int*>(base + ent_bytes + entr_bytes + cand_bytes);
            ba.cbound = reinterpret_cast<int*>(base + ent_bytes + entr_bytes + cand_bytes +
                                               (size_t)round_up(a.total_rows * kBandWarps * 4, 256));
            ba.counts = plane_counts;
            ba.Ws = lrWs;
            ba.H = (int)H;
            ba.W = (int)W;
            ba.Wp = Wp;
            ba.nb = band.nb;
            ba.Ww = (int)Ww;
            ba.n_img = band.n_img;
            ba.pol0 = band.pol0;
            ba.nplanes = (int)nimg;
            ba.band0 = 0;
            ba.Hg = (int)H;
            ba.group = bgroup;
            ba.ngroups = (int)ngroups;
            ba.pts_gate = a.pts_gate;
            ba.all_planes = false;
            const int rc = launch_band_path(a, ba, take_new, st);
            if (rc != DFC_OK) return rc;
        }
        if (anc_on) {
            RowArgs aa = a;
            aa.vec_nr = aligned(nr, 16) && Wp % 8 == 0 && a.nr_img_stride % 8 == 0;
            if (band.bmask && band.anc) {  // stage rows from the bands (no nr plane)
                aa.bmask = band.bmask;
                aa.babove = band.above;
                aa.bbelow = band.below;
            }
            const bool owners = LB != nullptr || NC != nullptr;
            const void* afn = take_new ? (owners ? anc_kernel_ptr<true, true>() : anc_kernel_ptr<true, false>())
                                       : (owners ? anc_kernel_ptr<false, true>() : anc_kernel_ptr<false, false>());
            const int asm_bytes = anc_smem_bytes((int)W);
            e = set_dyn_smem((const void*)(afn), asm_bytes);
            if (e != cudaSuccess) return cuda_fail(e);
            if (a.total_rows > 16384 && (a.pts_gate || a.lr_gate)) {
                // many rows, some owned by other kernels (C3: every plane a point
                // plane): a compact list first, so that skipped rows cost nothing
                const int64_t rblocks = std::min<int64_t>((a.total_rows + 255) / 256, 148 * 8);
                k_rows_rest<<<(unsigned)rblocks, 256, 0, os>>>(a.row_done, plane_counts, a.total_rows, (int)H,
                                                               (int)W, a.lr_gate, a.pts_gate, rest_rows, rest_count);
                ++g_launches;
                aa.row_list = rest_rows;
                aa.row_count = rest_count;
            }
            // one CTA per row (the block scheduler balances rows of unequal cost;
            // a grid-stride cap of 16 CTAs per SM left 27% of the slots idle on
            // the last round of rows: C2 row pass 0.320 -> 0.287 ms).  A compact
            // row list (count on the device) keeps the grid-stride cap.
            static const int anc_cap = [] {  // DFC_ANC_CAP (tuning): CTAs per SM, 0 = one CTA per row
                const char* v = getenv("DFC_ANC_CAP");
                return v ? atoi(v) : 0;
            }();
            const int64_t ablocks =
                (anc_cap <= 0 && !aa.row_list) ? a.total_rows : std::min<int64_t>(a.total_rows, 148 * (anc_cap > 0 ? anc_cap : 16));
            void* aargs[] = {&aa};
            e = cudaLaunchKernel(afn, dim3((unsigned)ablocks), dim3(32 * kAncWarps), aargs, (size_t)asm_bytes, os);
            if (e != cudaSuccess) return cuda_fail(e);
            ++g_launches;
            return DFC_OK;
        }
        // the segment kernel over the remaining rows: few rows -> one CTA group per
        // row group, skipping flagged rows (cheapest); many rows -> a compact
        // list first, so that skipped rows cost no CTA launch
        if (a.total_rows <= 16384) {
            void* args[] = {&a};
            e = cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(g.R * g.T), args, (size_t)g.smem_bytes, os);
            if (e != cudaSuccess) return cuda_fail(e);
            ++g_launches;
            return DFC_OK;
        }
        const int64_t rblocks = std::min<int64_t>((a.total_rows + 255) / 256, 148 * 8);
        k_rows_rest<<<(unsigned)rblocks, 256, 0, os>>>(a.row_done, plane_counts, a.total_rows, (int)H, (int)W,
                                                       a.lr_gate, a.pts_gate, rest_rows, rest_count);
        ++g_launches;
        RowArgs ra = a;
        ra.row_list = rest_rows;
        ra.row_count = rest_count;
        ra.row_done = nullptr;
        void* args[] = {&ra};
        const int64_t sblocks = std::min<int64_t>(blocks, 148 * 8);  // grid-stride over the list (often empty)
        e = cudaLaunchKernel(fn, dim3((unsigned)sblocks), dim3(g.R * g.T), args, (size_t)g.smem_bytes, os);
        if (e != cudaSuccess) return cuda_fail(e);
        ++g_launches;
        return DFC_OK;
    }

    void* args[] = {&a};
    e = cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(g.R * g.T), args, (size_t)g.smem_bytes, st);
    if (e != cudaSuccess) return cuda_fail(e);
    ++g_launches;
    return DFC_OK;
}

int64_t pstride(const void* a, const void* b) {
    return reinterpret_cast<const char*>(b) - reinterpret_cast<const char*>(a);
}

// Shared driver for dfc_edt_u8 / _dual / _batched.
int edt_core(const uint8_t* img, int64_t n, int64_t H, int64_t W, int64_t pitch, int64_t istride,
             int pol0, int npol, const OutSet& o, cudaStream_t st) {
    if (!img || !o.D[0] || (npol == 2 && !o.D[1])) return DFC_ERR_ARG;
    if (!shape_ok(H, W)) return DFC_ERR_SHAPE;
    if (pitch < W || n < 1 || n > 65535 || (n > 1 && istride < H * pitch)) return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    const int Wp = (int)round_up(W, 8);
    const int64_t nb = (H + kBand - 1) / kBand;
    const int64_t planes = (int64_t)npol * n;
    const size_t carry_elems = (size_t)(planes * nb * Wp);
    const size_t nr_elems = (size_t)(planes * H * Wp);
    // point planes (k_rows_pts) in the default row pass when planes are whole warps of rows
    const int mode = g_row_mode != 0 ? g_row_mode : env_row_mode();
    const bool pts_on = (mode == 4 || mode == 6) && H % 32 == 0;
    // band source: k_rows_anc stages the rows of the planes it owns from the
    // column pass's band masks and carries; K1c writes no nearest-row plane there
    // (single images: K1a writes the masks before the point-plane test is known,
    // which would cost batches of point planes, C3, a mask write per pixel / 8)
    const bool band_on = mode == 6 && anc_dense_on() && W <= kAncMaxW && H <= 32768 && n == 1;
    // band masks for every single image: K1c then builds the nearest-row plane
    // from them instead of re-reading the image (C5: 1 B/px of reads less)
    const bool masks_on = n == 1;
    // sparse planes of single images: the band path (k_rows_band.cu), no plane
    const bool sparse_band = mode == 6 && masks_on && band_sparse_on() && H * W >= band_min_px();
    const size_t bmask_elems = masks_on ? (size_t)(n * nb * Wp) : 0;
    Scratch sc(st);
    cudaError_t e = sc.alloc((2 * carry_elems + nr_elems) * sizeof(uint16_t) + 512 + (size_t)planes * 8 +
                             (pts_on ? (size_t)planes * kPtsCap * 4 : 0) + bmask_elems * 4 + 16);
    if (e != cudaSuccess) return cuda_fail(e);
    uint16_t* first = static_cast<uint16_t*>(sc.p);
    uint16_t* last = first + carry_elems;
    uint16_t* nr = reinterpret_cast<uint16_t*>(round_up(reinterpret_cast<uintptr_t>(last + carry_elems), 16));
    auto* counts = reinterpret_cast<unsigned long long*>(round_up(reinterpret_cast<uintptr_t>(nr + nr_elems), 16));
    uint32_t* pts = pts_on ? reinterpret_cast<uint32_t*>(counts + planes) : nullptr;
    uint32_t* bmask = masks_on ? reinterpret_cast<uint32_t*>(round_up(
                                    reinterpret_cast<uintptr_t>(reinterpret_cast<char*>(counts + planes) +
                                                                (pts_on ? (size_t)planes * kPtsCap * 4 : 0)), 16))
                              : nullptr;
    const int64_t Ww = (W + 31) / 32;
    Scratch so(st);  // object-column bits per (plane, band) for the band path's hull filter
    if (sparse_band) {
        e = so.alloc((size_t)(planes * nb * Ww) * 4);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    uint32_t* objcol = static_cast<uint32_t*>(so.p);
    prof(0, st);
    int rc = column_pass(img, n, H, W, pitch, istride, pol0, npol, nr, first, last, Wp, st, nullptr, counts, pts,
                         bmask, band_on, false, sparse_band, objcol);
    if (rc != DFC_OK) return rc;
    prof(1, st);

    // one launch per tie policy when every output is present for all planes
    // with a uniform stride; otherwise per plane
    const int64_t plane_bytes = H * W * 4;
    auto stride_of = [&](const void* p0, const void* p1) -> int64_t {
        return npol == 2 ? pstride(p0, p1) : plane_bytes;
    };
    bool uniform = true;
    if (npol == 2) {
        uniform = ((o.S[0] == nullptr) == (o.S[1] == nullptr)) &&
                  ((o.LB[0] == nullptr) == (o.LB[1] == nullptr)) &&
                  ((o.NC[0] == nullptr) == (o.NC[1] == nullptr));
    }
    const bool want_keep = o.D[0] || o.S[0] || o.LB[0];
    if (uniform) {
        const int64_t nimg = planes;
        BandSrc bs;
        bs.bmask = bmask;
        bs.anc = band_on;
        bs.sparse = sparse_band;
        bs.above = last;
        bs.below = first;
        bs.objcol = objcol;
        bs.nb = (int)nb;
        bs.n_img = (int)n;
        bs.pol0 = pol0;
        if (want_keep) {
            rc = row_pass(nr, nimg, H, W, Wp, false, o.D[0], stride_of(o.D[0], o.D[1]), o.S[0],
                          o.S[0] ? stride_of(o.S[0], o.S[1]) : 0, o.LB[0],
                          o.LB[0] ? stride_of(o.LB[0], o.LB[1]) : 0, nullptr, 0, st, false, 0, 0, 0, counts, pts, bs);
            if (rc != DFC_OK) return rc;
        }
        if (o.NC[0]) {
            rc = row_pass(nr, nimg, H, W, Wp, true, nullptr, 0, nullptr, 0, nullptr, 0, o.NC[0],
                          stride_of(o.NC[0], o.NC[1]), st, false, 0, 0, 0, counts, pts, bs);
            if (rc != DFC_OK) return rc;
        }
    } else {
        for (int s = 0; s < npol; ++s) {
            const uint16_t* pl = nr + (int64_t)s * H * Wp;
            BandSrc bs;  // n == 1 here
            bs.bmask = bmask;
            bs.anc = band_on;
            bs.sparse = sparse_band;
            bs.above = last + (int64_t)s * nb * Wp;
            bs.below = first + (int64_t)s * nb * Wp;
            bs.objcol = objcol ? objcol + (int64_t)s * nb * Ww : nullptr;
            bs.nb = (int)nb;
            bs.n_img = 1;
            bs.pol0 = pol0 + s;
            rc = row_pass(pl, 1, H, W, Wp, false, o.D[s], 0, o.S[s], 0, o.LB[s], 0, nullptr, 0, st, false, 0, 0, 0,
                          counts + s, pts ? pts + (int64_t)s * kPtsCap : nullptr, bs);
            if (rc != DFC_OK) return rc;
            if (o.NC[s]) {
                rc = row_pass(pl, 1, H, W, Wp, true, nullptr, 0, nullptr, 0, nullptr, 0, o.NC[s], 0, st, false, 0, 0,
                              0, counts + s, pts ? pts + (int64_t)s * kPtsCap : nullptr, bs);
                if (rc != DFC_OK) return rc;
            }
        }
    }
    prof(2, st);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e);
    return DFC_OK;
}

}  // namespace

extern "C" {

int dfc_edt_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes, int polarity,
               int32_t* d_sqdist, float* d_dist, int32_t* d_label, int32_t* d_nearest_col,
               dfc_stream_t stream) {
    if (polarity != DFC_BG_TO_OBJ && polarity != DFC_OBJ_TO_BG) return DFC_ERR_ARG;
    OutSet o;
    o.D[0] = d_sqdist;
    o.S[0] = d_dist;
    o.LB[0] = d_label;
    o.NC[0] = d_nearest_col;
    return edt_core(d_img, 1, rows, cols, pitch_bytes, 0, polarity, 1, o, (cudaStream_t)stream);
}

int dfc_edt_u8_dual(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                    int32_t* d_sqdist_bg, float* d_dist_bg, int32_t* d_sqdist_obj, float* d_dist_obj,
                    dfc_stream_t stream) {
    OutSet o;
    o.D[0] = d_sqdist_bg;
    o.D[1] = d_sqdist_obj;
    o.S[0] = d_dist_bg;
    o.S[1] = d_dist_obj;
    return edt_core(d_img, 1, rows, cols, pitch_bytes, 0, 0, 2, o, (cudaStream_t)stream);
}

int dfc_edt_u8_batched(const uint8_t* d_imgs, int64_t n, int64_t rows, int64_t cols,
                       int64_t pitch_bytes, int64_t image_stride_bytes, int32_t* d_sqdist,
                       float* d_dist, int32_t* d_label, dfc_stream_t stream) {
    OutSet o;
    o.D[0] = d_sqdist;
    o.S[0] = d_dist;
    o.LB[0] = d_label;
    return edt_core(d_imgs, n, rows, cols, pitch_bytes, image_stride_bytes, 0, 1, o,
                    (cudaStream_t)stream);
}

int dfc_vertical_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                    int32_t* d_vert, dfc_stream_t stream) {
    if (!d_img || !d_vert) return DFC_ERR_ARG;
    if (!shape_ok(rows, cols)) return DFC_ERR_SHAPE;
    if (pitch_bytes < cols) return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int Wp = (int)round_up(cols, 8);
    const int64_t nb = (rows + kBand - 1) / kBand;
    Scratch sc(st);
    cudaError_t e = sc.alloc(2 * (size_t)nb * Wp * sizeof(uint16_t));
    if (e != cudaSuccess) return cuda_fail(e);
    uint16_t* first = static_cast<uint16_t*>(sc.p);
    uint16_t* last = first + nb * Wp;
    column_pass(d_img, 1, rows, cols, pitch_bytes, 0, 0, 1, nullptr, first, last, Wp, st, d_vert);
    e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

namespace {
int vpass(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems, bool up, dfc_stream_t stream) {
    if (!d_map) return DFC_ERR_ARG;
    if (rows < 1 || cols < 1 || pitch_elems < cols) return DFC_ERR_ARG;
    g_launches = 0;
    const int64_t blocks = (cols + 255) / 256;
    if (blocks > 0x7fffffff) return DFC_ERR_SHAPE;
    if (up)
        k_vpass_u64<true><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_map, rows, cols, pitch_elems);
    else
        k_vpass_u64<false><<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_map, rows, cols, pitch_elems);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}
}  // namespace

int dfc_vertical_down_pass_u64(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems,
                               dfc_stream_t stream) {
    return vpass(d_map, rows, cols, pitch_elems, false, stream);
}

int dfc_vertical_up_pass_u64(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems,
                             dfc_stream_t stream) {
    return vpass(d_map, rows, cols, pitch_elems, true, stream);
}

int dfc_raster_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                  int32_t* d_cityblock, int32_t* d_chessboard, int32_t* d_chamfer34,
                  dfc_stream_t stream) {
    if (!d_img) return DFC_ERR_ARG;
    if (!shape_ok(rows, cols)) return DFC_ERR_SHAPE;
    if (pitch_bytes < cols) return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int Wp = (int)round_up(cols, 8);
    const int64_t nb = (rows + kBand - 1) / kBand;
    const size_t carry = (size_t)nb * Wp, nre = (size_t)rows * Wp;
    // anchored segments (k_raster_anc.cu) up to kRaMaxW columns, staging rows
    // from the band masks and carries; DFC_RASTER=window keeps the outward
    // window search (k_raster.cu) for A/B
    static const bool window = [] {
        const char* v = getenv("DFC_RASTER");
        return v && strcmp(v, "window") == 0;
    }();
    const bool anc = !window && cols <= kRaMaxW;
    Scratch sc(st);
    cudaError_t e = sc.alloc((2 * carry + (anc ? 0 : nre)) * sizeof(uint16_t) + 256 + (anc ? carry * 4 + 16 : 0));
    if (e != cudaSuccess) return cuda_fail(e);
    uint16_t* first = static_cast<uint16_t*>(sc.p);
    uint16_t* last = first + carry;
    uint16_t* nr = reinterpret_cast<uint16_t*>(round_up(reinterpret_cast<uintptr_t>(last + carry), 16));
    uint32_t* bmask = anc ? reinterpret_cast<uint32_t*>(nr) : nullptr;  // [nb][Wp] in place of the plane
    column_pass(d_img, 1, rows, cols, pitch_bytes, 0, 0, 1, anc ? nullptr : nr, first, last, Wp, st, nullptr,
                nullptr, nullptr, bmask, false, anc);
    RasterArgs r;
    r.nr = nr;
    r.Wp = Wp;
    r.H = (int)rows;
    r.W = (int)cols;
    r.T = 32;
    while (r.T < 1024 && (int64_t)r.T * 32 < cols) r.T <<= 1;
    r.L = 1;  // power of two: padded indices are a shift
    while ((int64_t)r.L * r.T < cols) r.L <<= 1;
    r.city = d_cityblock;
    r.chess = d_chessboard;
    r.cham = d_chamfer34;
    r.bmask = bmask;
    r.babove = last;
    r.bbelow = first;
    if (anc) {
        const bool p16 = rows <= kRa16MaxDim && cols <= kRa16MaxDim;
        const void* fn = p16 ? (const void*)k_raster_anc<true> : (const void*)k_raster_anc<false>;
        const int smem = ra_smem_bytes((int)cols, p16);
        e = set_dyn_smem((const void*)(fn), smem);
        if (e != cudaSuccess) return cuda_fail(e);
        static const int ra_cap = [] {  // DFC_RA_CAP (tuning): CTAs per SM, 0 = one CTA per row
            const char* v = getenv("DFC_RA_CAP");
            return v ? atoi(v) : 0;
        }();
        const int64_t blocks = ra_cap <= 0 ? rows : std::min<int64_t>(rows, 148 * ra_cap);
        void* args[] = {&r};
        e = cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(32 * kRaWarps), args, (size_t)smem, st);
        if (e != cudaSuccess) return cuda_fail(e);
    } else {
        const int padW = (int)(cols + cols / r.L + 1);
        const int smem = (2 * padW + 2 * r.T + 2) * 4;
        e = set_dyn_smem((const void*)(k_raster), smem);
        if (e != cudaSuccess) return cuda_fail(e);
        k_raster<<<(unsigned)rows, r.T, smem, st>>>(r);
    }
    ++g_launches;
    e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_label_ordinals(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                       const int32_t* d_label, uint32_t* d_ordinal, dfc_stream_t stream) {
    if (!d_img || !d_label || !d_ordinal) return DFC_ERR_ARG;
    if (!shape_ok(rows, cols)) return DFC_ERR_SHAPE;
    if (pitch_bytes < cols) return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int nw = (int)((cols + 31) / 32);
    Scratch sc(st);
    const size_t words = 2 * (size_t)rows * nw + 2 * (size_t)rows;
    cudaError_t e = sc.alloc(words * 4);
    if (e != cudaSuccess) return cuda_fail(e);
    uint32_t* masks = static_cast<uint32_t*>(sc.p);
    uint32_t* wpre = masks + rows * nw;
    uint32_t* rowcnt = wpre + rows * nw;
    uint32_t* rowbase = rowcnt + rows;
    k_ord_rows<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(d_img, pitch_bytes, (int)rows,
                                                                   (int)cols, nw, masks, wpre, rowcnt);
    k_ord_scan<<<1, 1024, 0, st>>>(rowcnt, rowbase, (int)rows);
    const int64_t n = rows * cols;
    k_ord_map<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(
        d_label, n, (int)cols, nw, masks, wpre, rowbase, d_ordinal);
    g_launches += 3;
    e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_column_nr_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes, int polarity,
                     uint16_t* d_nr, int64_t nr_pitch, dfc_stream_t stream) {
    if (!d_img || !d_nr || (polarity != 0 && polarity != 1)) return DFC_ERR_ARG;
    if (!shape_ok(rows, cols)) return DFC_ERR_SHAPE;
    if (pitch_bytes < cols || nr_pitch < round_up(cols, 4) || nr_pitch % 4 != 0 || !aligned(d_nr, 8))
        return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nb = (rows + kBand - 1) / kBand;
    Scratch sc(st);
    cudaError_t e = sc.alloc(2 * (size_t)nb * nr_pitch * sizeof(uint16_t));
    if (e != cudaSuccess) return cuda_fail(e);
    uint16_t* first = static_cast<uint16_t*>(sc.p);
    uint16_t* last = first + nb * nr_pitch;
    column_pass(d_img, 1, rows, cols, pitch_bytes, 0, polarity, 1, d_nr, first, last, (int)nr_pitch, st);
    e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_rows_from_nr_u16(const uint16_t* d_nr, int64_t rows, int64_t cols, int64_t row0, int64_t tile_cols,
                         int64_t tile_stride_elems, int take_new, int32_t* d_sqdist, float* d_dist,
                         int32_t* d_label, int32_t* d_nearest_col, dfc_stream_t stream) {
    if (!d_nr || (!d_sqdist && !d_dist && !d_label && !d_nearest_col)) return DFC_ERR_ARG;
    if (rows < 1 || cols < 1 || cols > kMaxRowCols || row0 < 0 || row0 + rows > 65535) return DFC_ERR_SHAPE;
    const int64_t hi = row0 + rows - 1;
    if (hi * hi + (cols - 1) * (cols - 1) > DFC_MAX_SQDIST) return DFC_ERR_SHAPE;
    if (tile_cols < 2 || tile_cols % 2 != 0 || !aligned(d_nr, 4) || tile_stride_elems % 2 != 0) return DFC_ERR_ARG;
    if (tile_cols < cols && tile_stride_elems < rows * tile_cols) return DFC_ERR_ARG;
    if (take_new && d_label) return DFC_ERR_ARG;  // labels follow the keep_old rule
    init_pool_once();
    g_launches = 0;
    prof(1, (cudaStream_t)stream);
    // object pixels of this row stripe (the per-plane kernel choice of row_pass)
    cudaStream_t st = (cudaStream_t)stream;
    Scratch cs(st);
    cudaError_t ce = cs.alloc(sizeof(unsigned long long));
    if (ce != cudaSuccess) return cuda_fail(ce);
    auto* counts = static_cast<unsigned long long*>(cs.p);
    ce = cudaMemsetAsync(counts, 0, sizeof(unsigned long long), st);
    if (ce != cudaSuccess) return cuda_fail(ce);
    {
        RowArgs ca{};
        ca.nr = d_nr;
        ca.Wp = (int)std::min<int64_t>(tile_cols, 1 << 30);
        ca.tile_cols = ca.Wp;
        ca.tile_stride = tile_stride_elems;
        ca.row0 = (int)row0;
        ca.H = (int)rows;
        ca.W = (int)cols;
        ca.total_rows = rows;
        k_nr_count<<<(unsigned)std::min<int64_t>(rows, 148 * 8), 256, 0, st>>>(ca, counts);
        ++g_launches;
    }
    const int rc = row_pass(d_nr, 1, rows, cols, (int)std::min<int64_t>(tile_cols, 1 << 30), take_new != 0,
                            d_sqdist, 0, d_dist, 0, d_label, 0, d_nearest_col, 0, st, false,
                            (int)std::min<int64_t>(tile_cols, 1 << 30), tile_stride_elems, (int)row0, counts);
    if (rc != DFC_OK) return rc;
    prof(2, (cudaStream_t)stream);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_envelope_vdist_u16(const uint16_t* d_vdist, int64_t rows, int64_t cols, int64_t pitch_elems,
                           int take_new, int32_t* d_sqdist, float* d_dist, int32_t* d_nearest_col,
                           dfc_stream_t stream) {
    if (!d_vdist || (!d_sqdist && !d_dist && !d_nearest_col)) return DFC_ERR_ARG;
    if (!shape_ok(rows, cols)) return DFC_ERR_SHAPE;
    if (pitch_elems < cols || pitch_elems % 2 != 0 || !aligned(d_vdist, 4)) return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    const int rc = row_pass(d_vdist, 1, rows, cols, (int)pitch_elems, take_new != 0, d_sqdist, 0, d_dist,
                            0, nullptr, 0, d_nearest_col, 0, (cudaStream_t)stream, true);
    if (rc != DFC_OK) return rc;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_sqrt_i32(const int32_t* d_sqdist, float* d_dist, int64_t n, dfc_stream_t stream) {
    if (!d_sqdist || !d_dist || n < 0) return DFC_ERR_ARG;
    g_launches = 0;
    if (n == 0) return DFC_OK;
    k_sqrt_i32<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, (cudaStream_t)stream>>>(
        d_sqdist, d_dist, n);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

static unsigned grid_for(int64_t n, int per_block = 256, int cap = 148 * 16) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + per_block - 1) / per_block, cap));
}

int dfc_unpack_pbm(const uint8_t* d_bits, int64_t rows, int64_t cols, int64_t row_bytes, int invert,
                   uint8_t* d_img, int64_t pitch_bytes, dfc_stream_t stream) {
    if (!d_bits || !d_img || rows < 1 || cols < 1 || row_bytes != (cols + 7) / 8 || pitch_bytes < cols)
        return DFC_ERR_ARG;
    g_launches = 0;
    k_unpack_pbm<<<grid_for(rows * row_bytes), 256, 0, (cudaStream_t)stream>>>(d_bits, rows, cols, row_bytes,
                                                                              invert, d_img, pitch_bytes);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_binarize_u8(const uint8_t* d_src, int64_t rows, int64_t cols, int64_t src_pitch, int invert,
                    uint8_t* d_dst, int64_t dst_pitch, dfc_stream_t stream) {
    if (!d_src || !d_dst || rows < 1 || cols < 1 || src_pitch < cols || dst_pitch < cols) return DFC_ERR_ARG;
    g_launches = 0;
    k_binarize<<<grid_for(rows * cols), 256, 0, (cudaStream_t)stream>>>(d_src, rows, cols, src_pitch, invert,
                                                                       d_dst, dst_pitch);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_count_objects_u8(const uint8_t* d_img, int64_t rows, int64_t cols, int64_t pitch_bytes,
                         uint64_t* d_count, dfc_stream_t stream) {
    if (!d_img || !d_count || rows < 1 || cols < 1 || pitch_bytes < cols) return DFC_ERR_ARG;
    g_launches = 0;
    k_count<<<grid_for(rows * cols), 256, 0, (cudaStream_t)stream>>>(
        d_img, rows, cols, pitch_bytes, reinterpret_cast<unsigned long long*>(d_count));
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_gray_i32(const int32_t* d_map, int64_t n, int mode, uint8_t* d_gray, int32_t* d_max,
                 uint32_t* d_scratch, dfc_stream_t stream) {
    if (!d_map || !d_gray || !d_max || !d_scratch || n < 1 || (mode != 0 && mode != 1)) return DFC_ERR_ARG;
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d_scratch, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return cuda_fail(e);
    k_max_finite<<<grid_for(n), 256, 0, st>>>(d_map, n, d_scratch);
    k_gray<<<grid_for(n), 256, 0, st>>>(d_map, n, mode, d_scratch, d_gray, d_max);
    g_launches += 2;
    e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_labels_gray(const uint32_t* d_ordinal, int64_t n, int64_t feature_count, uint8_t* d_gray,
                    dfc_stream_t stream) {
    if (!d_ordinal || !d_gray || n < 1) return DFC_ERR_ARG;
    if (feature_count < 1) return DFC_ERR_NO_FEATURES;
    g_launches = 0;
    k_labels_gray<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_ordinal, n, (double)feature_count, d_gray);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_row_owners_i64(const int64_t* d_vert, int64_t rows, int64_t cols, int64_t pitch_elems, int64_t lmax,
                       int take_new, int32_t* d_owner, int64_t* d_value, dfc_stream_t stream) {
    if (!d_vert || !d_owner || rows < 1 || cols < 1 || cols > 0x7fffffff || pitch_elems < cols) return DFC_ERR_ARG;
    g_launches = 0;
    const unsigned blocks = (unsigned)std::min<int64_t>(rows, 148 * 8);
    if (take_new)
        k_row_owners<true><<<blocks, 32 * kOwnWarps, 0, (cudaStream_t)stream>>>(d_vert, rows, (int)cols, pitch_elems,
                                                                              lmax, d_owner, d_value);
    else
        k_row_owners<false><<<blocks, 32 * kOwnWarps, 0, (cudaStream_t)stream>>>(d_vert, rows, (int)cols, pitch_elems,
                                                                               lmax, d_owner, d_value);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_raster_pass_u64(uint64_t* d_map, int64_t rows, int64_t cols, int64_t pitch_elems, int pass,
                        dfc_stream_t stream) {
    if (!d_map || rows < 1 || cols < 1 || pitch_elems < cols || pass < 0 || pass > 5) return DFC_ERR_ARG;
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    switch (pass) {
        case DFC_PASS_CITYBLOCK_FORWARD: k_raster_pass<<<1, 1024, 0, st>>>(d_map, rows, cols, pitch_elems, 0); break;
        case DFC_PASS_CITYBLOCK_BACKWARD: k_raster_pass<<<1, 1024, 0, st>>>(d_map, rows, cols, pitch_elems, 1); break;
        case DFC_PASS_CHAMFER_FORWARD: k_raster_pass<<<1, 1024, 0, st>>>(d_map, rows, cols, pitch_elems, 2); break;
        case DFC_PASS_CHAMFER_BACKWARD: k_raster_pass<<<1, 1024, 0, st>>>(d_map, rows, cols, pitch_elems, 3); break;
        case DFC_PASS_CITYBLOCK_VERTICAL:
            k_vpass_cb<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(d_map, rows, cols, pitch_elems);
            break;
        default:
            k_hpass_cb<<<(unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 16), 256, 0, st>>>(d_map, rows, cols,
                                                                                              pitch_elems);
    }
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_danielsson_u8(const uint8_t* d_img, int64_t n_images, int64_t rows, int64_t cols, int64_t pitch_bytes,
                      int64_t image_stride_bytes, int first_sweep_only, uint64_t* d_dist, uint32_t* d_dy,
                      uint32_t* d_dx, dfc_stream_t stream) {
    if (!d_img || !d_dist || !d_dy || !d_dx || n_images < 1 || n_images > 0x7fffffff) return DFC_ERR_ARG;
    if (rows < 1 || cols < 1 || rows > 65535 || cols > 65535) return DFC_ERR_SHAPE;
    if (pitch_bytes < cols || (n_images > 1 && image_stride_bytes < rows * pitch_bytes)) return DFC_ERR_ARG;
    init_pool_once();
    g_launches = 0;
    cudaStream_t st = (cudaStream_t)stream;
    DanArgs a;
    a.img = d_img;
    a.pitch = pitch_bytes;
    a.img_stride = image_stride_bytes;
    a.rows = (int)rows;
    a.cols = (int)cols;
    a.Wb = (int)round_up(cols, 2);
    a.first_only = first_sweep_only != 0;
    a.dist = d_dist;
    a.dy = d_dy;
    a.dx = d_dx;
    a.scratch = nullptr;
    const size_t smem = (size_t)2 * 16 * a.Wb;  // two rows of (uint64 D, uint32 dy, uint32 dx)
    Scratch sc(st);
    if (smem > 200 * 1024) {  // rows too wide for shared memory: the same layout in global scratch
        const cudaError_t e = sc.alloc(smem * (size_t)n_images);
        if (e != cudaSuccess) return cuda_fail(e);
        a.scratch = static_cast<char*>(sc.p);
    } else {
        const cudaError_t e = set_dyn_smem((const void*)k_danielsson, (int)smem);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    k_danielsson<<<(unsigned)n_images, kDanThreads, a.scratch ? 0 : smem, st>>>(a);
    ++g_launches;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DFC_OK : cuda_fail(e);
}

int dfc_set_profile_events(void* ev_col_begin, void* ev_row_begin, void* ev_row_end) {
    g_ev[0] = static_cast<cudaEvent_t>(ev_col_begin);
    g_ev[1] = static_cast<cudaEvent_t>(ev_row_begin);
    g_ev[2] = static_cast<cudaEvent_t>(ev_row_end);
    return DFC_OK;
}

int dfc_set_row_kernel(int mode) {
    if (mode < 0 || mode > 6 || mode == 2 || mode == 3) return DFC_ERR_ARG;  // 2, 3: retired kernels
    g_row_mode = mode;
    return DFC_OK;
}

int dfc_set_lr_chunk(int cols) {
    if (cols < 0 || cols % 32 != 0 || cols > 65536) return DFC_ERR_ARG;
    g_lr_chunk = cols;
    return DFC_OK;
}

int dfc_set_band_min_pixels(int64_t pixels) {
    g_band_min_px = pixels < 0 ? -1 : pixels;
    return DFC_OK;
}

int dfc_last_launch_count(void) { return g_launches; }

long long dfc_debug_guard_violations(void) {
    unsigned long long v = 0;
    if (cudaMemcpyFromSymbol(&v, g_guard_bad, sizeof(v)) != cudaSuccess) return -1;
    return guard_on() ? (long long)v : -1;
}

int dfc_last_cuda_error(void) { return g_last_cuda; }

const char* dfc_status_string(int status) {
    switch (status) {
        case DFC_OK: return "ok";
        case DFC_ERR_SHAPE: return "unsupported shape (rows/cols range or int32 distance bound)";
        case DFC_ERR_ARG: return "invalid argument";
        case DFC_ERR_CUDA: return "CUDA error";
        case DFC_ERR_NCCL: return "NCCL error";
        case DFC_ERR_NO_FEATURES: return "no features: voronoi labels undefined";
        default: return "unknown status";
    }
}

const char* dfc_version(void) { return "distfield-b200 0.1 sm_100a"; }

}  // extern "C"
