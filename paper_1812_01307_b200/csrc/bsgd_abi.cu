// C ABI of the B200-native BSGD-TV epoch path (declared in include/bsgd_b200.h).
//
// Owns the resident matrix (A as CSR and A^T as CSR, built on the device at
// plan creation), launches the SpMV / TV-prox kernels, and keeps every
// compute entry point stream-ordered and graph-capturable.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdlib>

#include "../../include/bsgd_b200.h"
#include "common.cuh"
#include "fgp.cuh"
#include "fgp2.h"
#include "spmv.cuh"
#include "siddon.cuh"
#include "stacked.cuh"
#include "gtile.cuh"
#include "slab.cuh"

using namespace bsgd;

#define BSGD_VERSION 111

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(e_ == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA,        \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                         \
    } while (0)

#define LAUNCHED()                                                                          \
    do {                                                                                    \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess)                                                              \
            return fail(BSGD_ECUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                \
    } while (0)

// ---------------------------------------------------------------------------
// device facts and occupancy (cached; queried outside graph capture first)
// ---------------------------------------------------------------------------
static std::mutex g_mu;
static std::unordered_map<const void *, int> g_occ;
static int g_sms[64];

static int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (g_sms[dev] == 0) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        g_sms[dev] = n > 0 ? n : kNumSMs;
    }
    return g_sms[dev];
}

template <typename K>
static int occupancy(K kernel) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find((const void *)kernel);
    if (it != g_occ.end()) return it->second;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, 0);
    if (nb < 1) nb = 1;
    g_occ[(const void *)kernel] = nb;
    return nb;
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

static inline int pow2_floor(int64_t v) {
    int p = 1;
    while ((int64_t)p * 2 <= v) p *= 2;
    return p;
}

// depth ds of numpy's pairwise recursion at which the first leaf (n <= 128)
// appears: the tree above it is a perfect binary tree (pairwise.cuh).  Also
// checks that every subtree below finishes within pw_node's 4 levels.
static int pw_depth(int64_t N, int *ds_out) {
    std::vector<int64_t> sizes{N};
    int d = 0;
    for (;;) {
        bool leaf = false;
        for (int64_t s : sizes) leaf = leaf || s <= 128;
        if (leaf) break;
        std::vector<int64_t> nxt;
        for (int64_t s : sizes) {
            const int64_t a = pw_split(s), b = s - a;
            for (int64_t c : {a, b})
                if (std::find(nxt.begin(), nxt.end(), c) == nxt.end()) nxt.push_back(c);
        }
        sizes.swap(nxt);
        ++d;
    }
    for (int64_t s : sizes) {  // levels still needed below depth d
        std::vector<int64_t> cur{s};
        int lev = 0;
        while (true) {
            bool all = true;
            std::vector<int64_t> nxt;
            for (int64_t c : cur)
                if (c > 128) { all = false; nxt.push_back(pw_split(c)); nxt.push_back(c - pw_split(c)); }
            if (all) break;
            cur.swap(nxt);
            if (++lev > 4) return fail(BSGD_EINVAL, "pairwise tree too deep for %lld elements", (long long)N);
        }
    }
    *ds_out = d;
    return BSGD_OK;
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct bsgd_plan {
    int device = 0;
    int64_t rows = 0, cols = 0, nnz = 0;
    int vdt = 8;
    int64_t M = 1, N = 1;
    std::vector<int64_t> row_bounds, col_bounds, block_nnz;
    int64_t *f_ptr = nullptr;
    int32_t *f_idx = nullptr;
    void *f_val = nullptr;
    int64_t *t_ptr = nullptr;
    int32_t *t_idx = nullptr;
    void *t_val = nullptr;
    int64_t *d_row_bounds = nullptr, *d_col_bounds = nullptr;
    int g_fwd = 32, g_tr = 32;
    size_t device_bytes = 0;
    // slice-stacked plans (stacked.cuh): A = A2 (x) I_depth in interleaved order;
    // f_* / t_* then hold A2 / A2^T and rows/cols/nnz above are the logical sizes
    int64_t depth = 1;
    int64_t srows = 0, scols = 0, snnz = 0;  // stored CSR (A itself, or A2)
    int lanes = 32, kz_fwd = 1, kz_tr = 1;
    int64_t *d_col_sbounds = nullptr, *d_row_sbounds = nullptr;  // bounds / depth when all are multiples of it
    // tile-staged copies of A2 / A2^T (stacked.cuh, stacked_tile_kernel), set by
    // bsgd_plan_stacked_tiles
    struct StkTileStore {
        bool ok = false;
        int64_t ntiles = 0;
        int64_t *tile_ptr = nullptr, *seg_ptr = nullptr, *seg_uni = nullptr, *seg_ent = nullptr;
        int32_t *tile_rows = nullptr, *seg_nj = nullptr, *uni = nullptr;
        uint16_t *seg_row = nullptr;
        void *ent = nullptr;
        int kz = 4;             // slices per consumer lane (stacked.cuh tile_seg / tile_zc)
        size_t bytes = 0;
    } sf, stt;
    // gather-tiled copies of A / A^T (gtile.cuh), set by bsgd_plan_gather_tiles
    struct GTileStore {
        bool ok = false;
        int64_t ntiles = 0;
        int max_union = 0;
        int64_t *tile_ptr = nullptr, *row_ptr = nullptr, *uni_ptr = nullptr;
        int32_t *tile_rows = nullptr, *uni = nullptr;
        uint16_t *loc = nullptr;
        void *val = nullptr;
        size_t bytes = 0;
    } gf, gt;
    // blocked copy of A's stream for long rows (spmv.cuh csr_blocked_kernel)
    struct BlkStore {
        bool ok = false;
        int gb = 32;            // lanes per row (blocks of 4 gb entries)
        int64_t *ptr = nullptr;
        int32_t *idx = nullptr;     // NULL when the compressed indices are used
        void *val = nullptr;
        int2 *half = nullptr;       // compressed indices (spmv.cuh blk_cols)
        uint16_t *off = nullptr;
        size_t bytes = 0;
        // column order of the stream (spmv.cuh blk_order_map): 0 = the matrix's own,
        // else the gathered vector's gh x gw grid (image pixels for A, the sinogram's
        // angles x bins for A^T) renumbered and the product gathers from xt, the
        // vector permuted the same way before each launch
        int order = 0;
        int gh = 0, gw = 0;
        double *xt = nullptr;
        int64_t nrows = 0, veclen = 0;
    } fb, tb;   // of A (built at plan creation for long rows), of A^T (bsgd_plan_blocked_transposed)
    bool stacked() const { return depth > 1; }
    // in-epoch phase timing (bsgd_plan_set_timing / bsgd_plan_timing): kPhaseEvents
    // events per eager bsgd_epoch on the launching stream, never inside a capture
    struct Timing {
        bool on = false;
        std::vector<cudaEvent_t> pool;
        size_t used = 0;
    };
    mutable Timing timing;
};

// phases: [0] K1(x_k) when the lookahead r is invalid, [1] K2 + step epilogue,
// [2] TV prox, [3] K1(x_next) lookahead, [4] tail
static constexpr int kPhaseEvents = BSGD_TIMING_PHASES + 1;

struct EpochTimer {
    cudaEvent_t *ev = nullptr;
    cudaStream_t st = nullptr;
    EpochTimer(const bsgd_plan *p, cudaStream_t s) : st(s) {
        bsgd_plan::Timing &T = p->timing;
        if (!T.on) return;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
            cudaGetLastError();
            return;
        }
        while (T.used + kPhaseEvents > T.pool.size()) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
            T.pool.push_back(e);
        }
        ev = &T.pool[T.used];
        T.used += kPhaseEvents;
        cudaEventRecord(ev[0], st);
    }
    void mark(int k) {
        if (ev) cudaEventRecord(ev[k], st);
    }
};

static void blk_free(bsgd_plan::BlkStore &b) {
    cudaFree(b.ptr); cudaFree(b.idx); cudaFree(b.val); cudaFree(b.half); cudaFree(b.off); cudaFree(b.xt);
    b = bsgd_plan::BlkStore();
}

static void gtiles_free(bsgd_plan::GTileStore &t) {
    cudaFree(t.tile_ptr); cudaFree(t.row_ptr); cudaFree(t.uni_ptr); cudaFree(t.tile_rows); cudaFree(t.uni);
    cudaFree(t.loc); cudaFree(t.val);
    t = bsgd_plan::GTileStore();
}

static void stk_tiles_free(bsgd_plan::StkTileStore &t) {
    cudaFree(t.tile_ptr); cudaFree(t.seg_ptr); cudaFree(t.seg_uni); cudaFree(t.seg_ent); cudaFree(t.tile_rows);
    cudaFree(t.seg_nj); cudaFree(t.uni); cudaFree(t.seg_row); cudaFree(t.ent);
    t = bsgd_plan::StkTileStore();
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

__global__ void check_csr_kernel(int64_t rows, int64_t cols, const int64_t *ptr, const int32_t *idx, int *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = ptr[r], e = ptr[r + 1];
        if (e < b) { atomicOr(bad, 1); continue; }
        int64_t prevc = -1;
        for (int64_t k = b; k < e; ++k) {
            const int64_t c = idx[k];
            if (c < 0 || c >= cols) { atomicOr(bad, 2); break; }
            if (c <= prevc) { atomicOr(bad, 4); break; }
            prevc = c;
        }
    }
}

__global__ void expand_rows_kernel(int64_t rows, const int64_t *ptr, int32_t *rowid) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) rowid[k] = (int32_t)r;
}

__global__ void iota_kernel(int64_t n, uint32_t *out) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = (uint32_t)k;
}

template <typename V>
__global__ void gather_transpose_kernel(int64_t nnz, const uint32_t *pos, const int32_t *rowid, const V *val,
                                        int32_t *t_idx, V *t_val) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = pos[k];
        t_idx[k] = rowid[p];
        t_val[k] = val[p];
    }
}

// t_ptr[c] = first position of key >= c in the sorted column keys
__global__ void col_ptr_kernel(int64_t cols, int64_t nnz, const uint32_t *keys, int64_t *t_ptr) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= cols; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if ((int64_t)keys[mid] < c) lo = mid + 1; else hi = mid;
        }
        t_ptr[c] = lo;
    }
}

__global__ void block_nnz_kernel(int64_t rows, const int64_t *ptr, const int32_t *idx, int64_t M,
                                 const int64_t *rb, int64_t N, const int64_t *cb, unsigned long long *cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = 0;
        while (i + 1 < M && rb[i + 1] <= r) ++i;
        int64_t lo = ptr[r];
        for (int64_t j = 0; j < N; ++j) {
            const int64_t hi = lower_bound_i32(idx, lo, ptr[r + 1], cb[j + 1]);
            if (hi > lo) atomicAdd(cnt + i * N + j, (unsigned long long)(hi - lo));
            lo = hi;
        }
    }
}

static void plan_free(bsgd_plan *p) {
    if (!p) return;
    DeviceGuard g(p->device);
    for (cudaEvent_t e : p->timing.pool) cudaEventDestroy(e);
    blk_free(p->fb);
    blk_free(p->tb);
    cudaFree(p->f_ptr); cudaFree(p->f_idx); cudaFree(p->f_val);
    cudaFree(p->t_ptr); cudaFree(p->t_idx); cudaFree(p->t_val);
    cudaFree(p->d_row_bounds); cudaFree(p->d_col_bounds);
    cudaFree(p->d_col_sbounds); cudaFree(p->d_row_sbounds);
    stk_tiles_free(p->sf);
    stk_tiles_free(p->stt);
    gtiles_free(p->gf);
    gtiles_free(p->gt);
    delete p;
}

static int grid_1d(int64_t n, int per_cta_items = kThreads) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, per_cta_items), (int64_t)num_sms() * 16));
}

template <typename V>
static int build_transpose(bsgd_plan *p, cudaStream_t st) {
    const int64_t nnz = p->snnz;
    int32_t *rowid = nullptr;
    uint32_t *keys_out = nullptr, *pos_in = nullptr, *pos_out = nullptr;
    void *temp = nullptr;
    size_t temp_bytes = 0;
    int rc = BSGD_OK;
    int end_bit = 1;
    while (end_bit < 32 && ((int64_t)1 << end_bit) <= p->scols) ++end_bit;
    auto cleanup = [&]() { cudaFree(rowid); cudaFree(keys_out); cudaFree(pos_in); cudaFree(pos_out); cudaFree(temp); };
#define TRY(call)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            rc = fail(e_ == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA,        \
                      "%s failed: %s", #call, cudaGetErrorString(e_));                   \
            cleanup();                                                                   \
            return rc;                                                                   \
        }                                                                                \
    } while (0)
    TRY(cudaMalloc(&rowid, sizeof(int32_t) * nnz));
    TRY(cudaMalloc(&keys_out, sizeof(uint32_t) * nnz));
    TRY(cudaMalloc(&pos_in, sizeof(uint32_t) * nnz));
    TRY(cudaMalloc(&pos_out, sizeof(uint32_t) * nnz));
    expand_rows_kernel<<<grid_1d(p->srows), kThreads, 0, st>>>(p->srows, p->f_ptr, rowid);
    iota_kernel<<<grid_1d(nnz), kThreads, 0, st>>>(nnz, pos_in);
    TRY(cudaGetLastError());
    const uint32_t *keys_in = reinterpret_cast<const uint32_t *>(p->f_idx);
    TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys_in, keys_out, pos_in, pos_out, nnz, 0,
                                        end_bit, st));
    TRY(cudaMalloc(&temp, temp_bytes));
    TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, pos_in, pos_out, nnz, 0,
                                        end_bit, st));
    gather_transpose_kernel<V><<<grid_1d(nnz), kThreads, 0, st>>>(nnz, pos_out, rowid, (const V *)p->f_val,
                                                                  p->t_idx, (V *)p->t_val);
    col_ptr_kernel<<<grid_1d(p->scols + 1), kThreads, 0, st>>>(p->scols, nnz, keys_out, p->t_ptr);
    TRY(cudaGetLastError());
    TRY(cudaStreamSynchronize(st));
#undef TRY
    cleanup();
    return BSGD_OK;
}


// Blocked copy of a stream (csr_blocked_kernel) of A (tr = false) or A^T (tr = true).
// (gh, gw) is the grid the gathered vector is laid out on (row-major, gh * gw = its
// length; 0, 0 = unknown): image pixels for A, the sinogram's angles x bins for A^T.
// Skipped quietly when memory is short.
template <typename V>
static int build_blocked_dir(bsgd_plan *p, bool tr, int gh, int gw, cudaStream_t st) {
    bsgd_plan::BlkStore b;
    b.nrows = tr ? p->cols : p->rows;
    b.veclen = tr ? p->rows : p->cols;
    const int64_t *sptr = tr ? p->t_ptr : p->f_ptr;
    const int32_t *sidx = tr ? p->t_idx : p->f_idx;
    const V *sval = (const V *)(tr ? p->t_val : p->f_val);
    // Gather order: a gh x gw grid is read in 4 x 4 tiles, one 128-byte line each, so a
    // row's consecutive entries (a ray's pixels; a pixel's bins over consecutive angles)
    // and the neighbouring rows of a warp share lines; the stream's entries keep their
    // positions (same sums, bit for bit) and the product gathers from the vector
    // permuted into that order (blk_order_map).  BSGD_BLK_ORDER = native | morton
    // overrides (experiments).
    int order = 1;
    if (const char *o = getenv("BSGD_BLK_ORDER"))
        order = strcmp(o, "tile4") == 0 ? 1 : strcmp(o, "morton") == 0 ? 2 : 0;
    if (gh <= 0 || gw <= 0 || (int64_t)gh * gw != b.veclen) order = 0;
    if (order == 2 && (gh != gw || (gw & (gw - 1)) != 0)) order = 0;
    // Tile shape (structural, from the matrix alone): the footprint of a gather
    // instruction -- 16 consecutive entries of a row -- on the grid.  Rays cross the
    // image in every direction (row and column spans balance: 4 x 4 tiles); a pixel's
    // entries run along the sinogram's angles with a slowly drifting bin (row spans
    // twice the column spans: 8 x 2 tiles, configs[3] K2 2.46-2.50 -> 2.24-2.29 ms once the
    // 64-warp build had made it L1-bound).  BSGD_BLK_TILE = 1 | 4 | 5 forces a shape.
    if (order == 1) {
        unsigned long long *acc = nullptr, h[3] = {0, 0, 0};
        if (cudaMalloc(&acc, sizeof(h)) == cudaSuccess) {
            cudaMemsetAsync(acc, 0, sizeof(h), st);
            blk_span_kernel<<<grid_1d(b.nrows, kThreads / 32), kThreads, 0, st>>>(b.nrows, sptr, sidx, gw, acc);
            cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            cudaFree(acc);
        }
        cudaGetLastError();
        if (h[2] > 0 && 2 * h[0] >= 3 * h[1]) order = 4;        // grid-row spans >= 1.5 x column spans
        else if (h[2] > 0 && 2 * h[1] >= 3 * h[0]) order = 5;
        if (const char *t = getenv("BSGD_BLK_TILE")) {
            const int v = atoi(t);
            if (v == 1 || v == 4 || v == 5) order = v;
        }
    }
    int64_t xt_len = b.veclen;
    if (order == 1) xt_len = (int64_t)((gh + 3) / 4) * ((gw + 3) / 4) * 16;
    if (order == 4) xt_len = (int64_t)((gh + 7) / 8) * ((gw + 1) / 2) * 16;
    if (order == 5) xt_len = (int64_t)((gh + 1) / 2) * ((gw + 7) / 8) * 16;
    if (xt_len > INT32_MAX) order = 0;
    // Lanes per row.  In the matrix's own column order, few lanes per ray and several
    // adjacent rays per warp: the neighbouring bins of a steep ray read the same sectors
    // in the same gather instruction (K1 at configs[3], ~920 nnz/row, round 1: 32 lanes
    // 4.03 ms, 16: 3.57, 8: 3.18, 4: 3.03; configs[2], ~460: 0.490 / 0.461 / 0.456 / 0.501).
    // In tile order a row's own consecutive entries share lines, the kernel is no longer
    // bound by L1 tag lookups (ncu: L1tex 96% -> 68%) and 16 lanes with the compressed
    // indices stream best (configs[3]: 4 lanes plain 3.01 ms, 8 compressed 2.56, 16
    // compressed 2.46, 32 plain 3.07; configs[2]: 8 -> 16 lanes 0.369 -> 0.317).
    const double mean = (double)p->nnz / (double)std::max<int64_t>(b.nrows, 1);
    // A^T in its own order (pixel rows of a CT system whose sinogram grid is unknown):
    // 8 lanes with compressed indices (configs[3] K2: 4 lanes plain 3.53 ms, 8 compressed
    // 3.29, 16: 3.83, 32: 5.60; the CSR kernel 6.1)
    b.gb = order ? 16 : tr ? 8 : mean >= 768.0 ? 4 : 8;
    if (const char *g = getenv(tr ? "BSGD_BLK_G_TR" : "BSGD_BLK_G")) {   // experiments
        const int v = atoi(g);
        if (v == 4 || v == 8 || v == 16 || v == 32) b.gb = v;
    }
    void *temp = nullptr;
    size_t temp_bytes = 0;
    int64_t total = 0;
    auto bail = [&](cudaError_t e) -> int {
        cudaGetLastError();
        cudaFree(temp);
        blk_free(b);
        if (e == cudaErrorMemoryAllocation) return BSGD_OK;   // keep the unblocked kernel
        return fail(BSGD_ECUDA, "blocked stream build failed: %s", cudaGetErrorString(e));
    };
    cudaError_t e = cudaMalloc(&b.ptr, sizeof(int64_t) * (b.nrows + 1));
    if (e != cudaSuccess) return bail(e);
    blk_len_kernel<<<grid_1d(b.nrows), kThreads, 0, st>>>(b.nrows, sptr, 4 * b.gb, b.ptr);
    e = cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, b.ptr, b.ptr, b.nrows + 1, st);
    if (e == cudaSuccess) e = cudaMalloc(&temp, temp_bytes);
    if (e == cudaSuccess) e = cudaMemsetAsync(b.ptr + b.nrows, 0, sizeof(int64_t), st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, b.ptr, b.ptr, b.nrows + 1, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&total, b.ptr + b.nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return bail(e);
    cudaFree(temp);
    temp = nullptr;
    e = cudaMalloc(&b.idx, sizeof(int32_t) * std::max<int64_t>(total, 1));
    if (e == cudaSuccess) e = cudaMalloc(&b.val, sizeof(V) * std::max<int64_t>(total, 1));
    if (e != cudaSuccess) return bail(e);
    blk_fill_kernel<V><<<grid_1d(b.nrows, kThreads / 32), kThreads, 0, st>>>(b.nrows, sptr, sidx, sval, b.ptr, b.idx,
                                                                             (V *)b.val, b.gb);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return bail(e);
    b.bytes = sizeof(int64_t) * (b.nrows + 1) + (sizeof(int32_t) + sizeof(V)) * (size_t)total;
    if (order) {
        e = cudaMalloc(&b.xt, sizeof(double) * xt_len);
        if (e == cudaSuccess) e = cudaMemsetAsync(b.xt, 0, sizeof(double) * xt_len, st);
        if (e != cudaSuccess) return bail(e);
        blk_renumber_kernel<<<grid_1d(total), kThreads, 0, st>>>(total, b.idx, gw, order);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return bail(e);
        b.order = order;
        b.gh = gh;
        b.gw = gw;
        b.bytes += sizeof(double) * xt_len;
    }
    // 16-bit column offsets from two bases per block when they fit (CT rays: the 2 gb
    // consecutive pixels of half a block lie a few image rows apart): 6 + 8 / (4 gb)
    // instead of 8 stream bytes per float32 entry
    if (!getenv("BSGD_NO_BLK_COMPRESS") && total > 0) {
        int2 *hh = nullptr;
        uint16_t *oo = nullptr;
        int *bad = nullptr;
        const int64_t nblocks = total / (4 * b.gb);
        cudaError_t e2 = cudaMalloc(&hh, sizeof(int2) * nblocks);
        if (e2 == cudaSuccess) e2 = cudaMalloc(&oo, sizeof(uint16_t) * total);
        if (e2 == cudaSuccess) e2 = cudaMalloc(&bad, sizeof(int));
        int hbad = 1;
        if (e2 == cudaSuccess) e2 = cudaMemsetAsync(bad, 0, sizeof(int), st);
        if (e2 == cudaSuccess) {
            blk_compress_kernel<<<grid_1d(nblocks), kThreads, 0, st>>>(nblocks, b.gb, b.idx, hh, oo, bad);
            e2 = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
        }
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(st);
        cudaFree(bad);
        if (e2 == cudaSuccess && hbad == 0) {   // both forms kept until tune_blocked picks one
            b.half = hh;
            b.off = oo;
            b.bytes += sizeof(uint16_t) * (size_t)total + sizeof(int2) * (size_t)nblocks;
        } else {
            cudaGetLastError();
            cudaFree(hh);
            cudaFree(oo);
        }
    }
    b.ok = true;
    bsgd_plan::BlkStore &dst = tr ? p->tb : p->fb;
    p->device_bytes -= dst.bytes;
    blk_free(dst);
    dst = b;
    p->device_bytes += b.bytes;
    return BSGD_OK;
}

// Grid of a gathered vector, inferred from the matrix alone (a plain CSR carries no
// geometry): the gaps between consecutive entries of a row peak at the grid width w (a
// pixel meets adjacent bins of one angle, then the next angle ~w rays further; a ray meets
// adjacent pixels of one image row, then the next row ~w pixels further), and w divides
// the vector's length.  Only the ORDER of the gathers depends on the answer -- the stream's
// entries keep their positions and the sums their bits -- so a wrong guess can cost time,
// never correctness.  Returns false when no width within 4 of the peak divides the rows
// or the peak holds less than 80% of the gaps.  BSGD_NO_GRID_INFER=1 disables it.
static bool infer_grid(const bsgd_plan *p, bool tr, cudaStream_t st, int *gh, int *gw) {
    // tr: A^T's rows gather from A's row space; else A's rows gather from its column space
    const int64_t srows = tr ? p->cols : p->rows, veclen = tr ? p->rows : p->cols;
    const int64_t *sptr = tr ? p->t_ptr : p->f_ptr;
    const int32_t *sidx = tr ? p->t_idx : p->f_idx;
    if (getenv("BSGD_NO_GRID_INFER") || srows < 1 || veclen < 64) return false;
    const int nbins = (int)std::min<int64_t>(veclen, 1 << 20);
    unsigned int *d_hist = nullptr;
    if (cudaMalloc(&d_hist, sizeof(unsigned int) * nbins) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    std::vector<unsigned int> hist(nbins);
    const int64_t stride = std::max<int64_t>(1, srows / 16384);   // ~16K sampled rows
    cudaMemsetAsync(d_hist, 0, sizeof(unsigned int) * nbins, st);
    blk_gap_hist_kernel<<<grid_1d(cdiv(srows, stride), kThreads / 32), kThreads, 0, st>>>(srows, stride, sptr, sidx,
                                                                                        nbins, d_hist);
    cudaMemcpyAsync(hist.data(), d_hist, sizeof(unsigned int) * nbins, cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d_hist);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    int64_t total = 0, peak = 0;
    for (int d = 2; d < nbins; ++d) {
        total += hist[d];
        if (hist[d] > hist[peak]) peak = d;
    }
    if (peak < 8 || total == 0) return false;
    int64_t best = 0;
    for (int64_t c = std::max<int64_t>(8, peak - 4); c <= std::min<int64_t>(nbins - 1, peak + 4); ++c)
        if (veclen % c == 0 && (best == 0 || std::llabs(c - peak) < std::llabs(best - peak))) best = c;
    if (best == 0 || veclen / best > INT32_MAX) return false;
    int64_t near = 0;
    for (int64_t d = std::max<int64_t>(2, best - 4); d <= std::min<int64_t>(nbins - 1, best + 4); ++d) near += hist[d];
    if (5 * near < 4 * total) return false;
    *gw = (int)best;
    *gh = (int)(veclen / best);
    return true;
}

// The forward copy is built at plan creation for plans whose rows are long (>= 384
// nonzeros on average: CT rays; padding to whole blocks then costs a few percent more
// stream bytes); a square column space is taken for an image (n x n, gathered in tile
// order).  BSGD_BLOCKED=force builds it for any plan (tests), BSGD_NO_BLOCKED=1 never.
template <typename V>
static int build_blocked(bsgd_plan *p, cudaStream_t st) {
    const char *force = getenv("BSGD_BLOCKED");
    const bool forced = force && strcmp(force, "force") == 0;
    if (p->stacked() || p->rows == 0 || getenv("BSGD_NO_BLOCKED") ||
        ((p->g_fwd != 32 || (double)p->nnz / (double)p->rows < 384.0) && !forced))
        return BSGD_OK;
    int img = (int)llround(sqrt((double)p->cols));
    if ((int64_t)img * img != p->cols || img % 4 != 0) img = 0;
    int gh = img, gw = img;
    if (!img && !infer_grid(p, false, st, &gh, &gw)) gh = gw = 0;   // a non-square image: width from the rays' index gaps
    return build_blocked_dir<V>(p, false, gh, gw, st);
}

// ---------------------------------------------------------------------------
// SpMV launchers
// ---------------------------------------------------------------------------
template <typename V>
static Csr<V> fwd_csr(const bsgd_plan *p, const double *vec) {
    return Csr<V>{p->rows, p->f_ptr, p->f_idx, (const V *)p->f_val, vec};
}
template <typename V>
static Csr<V> tr_csr(const bsgd_plan *p, const double *vec) {
    return Csr<V>{p->cols, p->t_ptr, p->t_idx, (const V *)p->t_val, vec};
}

static int ctas_for(int64_t nrows, int G, int cap) {
    const int64_t warps = cdiv(nrows, 32 / G);
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(warps, kThreads / 32), cap));
}

template <typename V, int GA, int GB, class EA, class EB>
static int launch_dual(const Csr<V> &A, const EA &ea, double *partA, int64_t *cntA, int64_t nnzA,
                       const Csr<V> &B, const EB &eb, double *partB, int64_t *cntB, int64_t nnzB,
                       cudaStream_t st) {
    auto kern = dual_csr_kernel<V, GA, GB, EA, EB>;
    const int cap = std::min(occupancy(kern) * num_sms(), kMaxPartials);
    const bool hasB = !std::is_same<EB, EpiNone>::value && B.nrows > 0;
    int nA = 0, nB = 0;
    if (hasB) {
        const double fa = (double)(nnzA + A.nrows) / (double)(nnzA + A.nrows + nnzB + B.nrows);
        const int capA = std::max(1, (int)std::lround(cap * fa));
        const int capB = std::max(1, cap - capA);
        nA = A.nrows > 0 ? ctas_for(A.nrows, GA, capA) : 0;
        nB = ctas_for(B.nrows, GB, capB);
    } else {
        nA = A.nrows > 0 ? ctas_for(A.nrows, GA, cap) : 0;
    }
    if (nA + nB == 0) return BSGD_OK;
    kern<<<nA + nB, kThreads, 0, st>>>(A, ea, partA, nA, cntA, B, eb, partB, cntB);
    LAUNCHED();
    return BSGD_OK;
}

// single product of one operand with lanes-per-row G chosen from the plan
template <typename V, class E>
static int launch_one(const Csr<V> &A, int G, const E &e, double *part, int64_t *cnt, int64_t nnz,
                      cudaStream_t st) {
    const Csr<V> none{0, nullptr, nullptr, nullptr, nullptr};
    if (G == 8) return launch_dual<V, 8, 8, E, EpiNone>(A, e, part, cnt, nnz, none, EpiNone{}, nullptr, nullptr, 0, st);
    if (G == 4) return launch_dual<V, 4, 8, E, EpiNone>(A, e, part, cnt, nnz, none, EpiNone{}, nullptr, nullptr, 0, st);
    return launch_dual<V, 32, 8, E, EpiNone>(A, e, part, cnt, nnz, none, EpiNone{}, nullptr, nullptr, 0, st);
}

// slice-stacked products (stacked.cuh).  EpiResid becomes the in-kernel
// y - z_0 - z_1 - ... chain with a plain store epilogue.
template <typename V, int KZ, bool RESID, bool ALIGNED, bool W, class E>
static int launch_stacked_k(const Stk<V> &A, const E &e, double *part, int64_t *cnt, cudaStream_t st) {
    auto kern = stacked_kernel<V, KZ, RESID, ALIGNED, W, E>;
    const int rpw = 32 / A.L;
    const int64_t items = cdiv(A.nrows, rpw) * cdiv(A.D, (int64_t)A.L * KZ);
    const int cap = std::min(occupancy(kern) * num_sms(), kMaxPartials);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(items, kThreads / 32), cap));
    kern<<<grid, kThreads, 0, st>>>(A, e, part, cnt);
    LAUNCHED();
    return BSGD_OK;
}

template <typename V, int KZ, bool RESID, class E>
static int launch_stacked_kz(const Stk<V> &A, const E &e, double *part, int64_t *cnt, cudaStream_t st) {
    const bool aligned = A.sbounds != nullptr;
    const bool wide = A.L == 32 && A.D % (32 * KZ) == 0;
    if (aligned && wide) return launch_stacked_k<V, KZ, RESID, true, true>(A, e, part, cnt, st);
    if (wide) return launch_stacked_k<V, KZ, RESID, false, true>(A, e, part, cnt, st);
    if (aligned) return launch_stacked_k<V, KZ, RESID, true, false>(A, e, part, cnt, st);
    return launch_stacked_k<V, KZ, RESID, false, false>(A, e, part, cnt, st);
}

template <typename V, bool RESID, class E>
static int launch_stacked(const Stk<V> &A, int kz, const E &e, double *part, int64_t *cnt, cudaStream_t st) {
    switch (kz) {
        case 4: return launch_stacked_kz<V, 4, RESID>(A, e, part, cnt, st);
        case 2: return launch_stacked_kz<V, 2, RESID>(A, e, part, cnt, st);
        default: return launch_stacked_kz<V, 1, RESID>(A, e, part, cnt, st);
    }
}

template <typename V, int KZ, bool RESID, bool ALIGNED, class E>
static int launch_stk_tile_kz(const Stk<V> &A, const bsgd_plan::StkTileStore &S, const E &e, double *part,
                              int64_t *cnt, cudaStream_t st) {
    auto kern = stacked_tile_kernel<V, KZ, RESID, ALIGNED, E>;
    const size_t smem = stk_tile_smem<V, KZ>();
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set = true;
    }
    StkTiles T{S.ntiles, S.tile_ptr, S.tile_rows, S.seg_ptr, S.seg_nj, S.seg_ent, S.seg_row, S.uni, S.ent};
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStkTileThreads, smem);
    const int64_t items = S.ntiles * (A.D / tile_zc<KZ>());
    const int cap = std::min(std::max(occ, 1) * num_sms(), kMaxPartials);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(items, cap));
    kern<<<grid, kStkTileThreads, smem, st>>>(A, T, e, part, cnt);
    LAUNCHED();
    return BSGD_OK;
}

template <typename V, bool RESID, bool ALIGNED, class E>
static int launch_stk_tile(const Stk<V> &A, const bsgd_plan::StkTileStore &S, const E &e, double *part, int64_t *cnt,
                           cudaStream_t st) {
    if (S.kz == 8) return launch_stk_tile_kz<V, 8, RESID, ALIGNED, E>(A, S, e, part, cnt, st);
    return launch_stk_tile_kz<V, 4, RESID, ALIGNED, E>(A, S, e, part, cnt, st);
}

static bool stk_tiles_used(const bsgd_plan *p, const bsgd_plan::StkTileStore &S) {
    return S.ok && p->depth % (32 * S.kz) == 0 && !getenv("BSGD_NO_STK_TILES");
}

template <typename V, class E>
static int launch_stacked_dir(const bsgd_plan *p, bool transposed, const double *vec, const E &e, double *part,
                              int64_t *cnt, cudaStream_t st) {
    Stk<V> A;
    A.nrows = transposed ? p->scols : p->srows;
    A.ptr = transposed ? p->t_ptr : p->f_ptr;
    A.idx = transposed ? p->t_idx : p->f_idx;
    A.val = (const V *)(transposed ? p->t_val : p->f_val);
    A.vec = vec;
    A.D = p->depth;
    A.bounds = transposed ? p->d_row_bounds : p->d_col_bounds;
    A.sbounds = transposed ? p->d_row_sbounds : p->d_col_sbounds;
    A.nb = transposed ? p->M : p->N;
    A.y = nullptr;
    A.L = p->lanes;
    const int kz = transposed ? p->kz_tr : p->kz_fwd;
    const bsgd_plan::StkTileStore &S = transposed ? p->stt : p->sf;
    if (stk_tiles_used(p, S)) {
        if constexpr (std::is_same<E, EpiResid>::value) {
            A.y = e.y;
            return A.sbounds ? launch_stk_tile<V, true, true>(A, S, EpiResidFinal{e.r}, part, cnt, st)
                             : launch_stk_tile<V, true, false>(A, S, EpiResidFinal{e.r}, part, cnt, st);
        } else {
            return A.sbounds ? launch_stk_tile<V, false, true>(A, S, e, part, cnt, st)
                             : launch_stk_tile<V, false, false>(A, S, e, part, cnt, st);
        }
    }
    if constexpr (std::is_same<E, EpiResid>::value) {
        A.y = e.y;
        return launch_stacked<V, true>(A, kz, EpiResidFinal{e.r}, part, cnt, st);
    } else {
        return launch_stacked<V, false>(A, kz, e, part, cnt, st);
    }
}

template <typename V, bool DB, class E>
static int launch_gtile_k(const bsgd_plan::GTileStore &S, const double *vec, const E &e, double *part, int64_t *cnt,
                          cudaStream_t st) {
    auto kern = gtile_kernel<V, DB, E>;
    const size_t smem = (DB ? 2 : 1) * sizeof(double) * (size_t)std::max(S.max_union, 1);
    static int attr_smem = 0;  // per instantiation
    if (attr_smem < (int)smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_smem = (int)smem;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    const int cap = std::min(std::max(occ, 1) * num_sms(), kMaxPartials);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(S.ntiles, cap));
    GTiles T{S.ntiles, S.tile_ptr, S.tile_rows, S.row_ptr, S.loc, S.val, S.uni_ptr, S.uni, S.max_union};
    kern<<<grid, kThreads, smem, st>>>(T, vec, e, part, cnt);
    LAUNCHED();
    return BSGD_OK;
}

// double-buffered windows while two of them fit three CTAs per SM
template <typename V, class E>
static int launch_gtile(const bsgd_plan::GTileStore &S, const double *vec, const E &e, double *part, int64_t *cnt,
                        cudaStream_t st) {
    if (2 * sizeof(double) * (size_t)S.max_union <= 72 * 1024) return launch_gtile_k<V, true>(S, vec, e, part, cnt, st);
    return launch_gtile_k<V, false>(S, vec, e, part, cnt, st);
}

static bool gtiles_on(const bsgd_plan::GTileStore &S) { return S.ok; }

template <typename V, class E>
static int launch_blocked(const bsgd_plan::BlkStore &B, bool tr, const double *vec, const E &e, double *part,
                          int64_t *cnt, cudaStream_t st) {
    if (B.order) {
        blk_permute_kernel<<<grid_1d(B.veclen), kThreads, 0, st>>>(B.veclen, vec, B.xt, B.gw, B.order);
        vec = B.xt;
    }
    CsrB<V> A{B.nrows, B.ptr, B.idx, (const V *)B.val, vec};
    A.half = B.half;
    A.off = B.off;
    auto go = [&](auto kern, int G) {
        const int cap = std::min(occupancy(kern) * num_sms(), kMaxPartials);
        kern<<<ctas_for(B.nrows, G, cap), kThreads, 0, st>>>(A, e, part, cnt);
    };
    const bool cmp = B.half != nullptr;
    // 16 lanes, compressed, tile order: A^T's pixel rows (twice as long as the rays, a
    // higher L1 hit rate) run best at 32 registers / 64 warps per SM, A's rays at 40 / 48
    // (configs[3]: K2 2.55-2.60 -> 2.47 ms, K1 2.42-2.46 -> 2.53 ms with 64 warps)
    static const int minb_tr = getenv("BSGD_BLK_MINB_TR") ? atoi(getenv("BSGD_BLK_MINB_TR")) : 8;   // experiments
    if (tr && B.gb == 16 && cmp && B.order && minb_tr == 8) go(csr_blocked_w64_kernel<V, 16, E, true>, 16);
    else if (B.gb == 16) cmp ? go(csr_blocked_kernel<V, 16, E, true>, 16) : go(csr_blocked_kernel<V, 16, E>, 16);
    else if (B.gb == 8) cmp ? go(csr_blocked_kernel<V, 8, E, true>, 8) : go(csr_blocked_kernel<V, 8, E>, 8);
    else if (B.gb == 4) cmp ? go(csr_blocked_kernel<V, 4, E, true>, 4) : go(csr_blocked_kernel<V, 4, E>, 4);
    else cmp ? go(csr_blocked_kernel<V, 32, E, true>, 32) : go(csr_blocked_kernel<V, 32, E>, 32);
    LAUNCHED();
    return BSGD_OK;
}

// Keep the compressed or the plain indices of the blocked copy by a fixed
// structural rule, so the kernel a plan runs does not depend on a timing race:
// compressed at 8 or more lanes per ray, plain at 4 (measured with A's own column
// order: configs[2], 8 lanes, 0.457 -> 0.415 ms compressed; configs[3], 4 lanes,
// 3.01 ms plain vs 3.07 compressed: the extra loads cost more than the bytes they
// save when the kernel is bound by L1 tag lookups).  BSGD_BLK_COMPRESS =
// force | off overrides the rule (tests run both variants against the oracle).
template <typename V>
static int tune_blocked(bsgd_plan *p, bsgd_plan::BlkStore &b) {
    if (!b.ok || b.half == nullptr || b.idx == nullptr) return BSGD_OK;
    bool keep_cmp = b.gb >= 8;
    if (const char *f = getenv("BSGD_BLK_COMPRESS")) {
        if (strcmp(f, "force") == 0) keep_cmp = true;
        else if (strcmp(f, "off") == 0) keep_cmp = false;
    }
    if (keep_cmp) {
        cudaFree(b.idx);
        b.idx = nullptr;
    } else {
        cudaFree(b.half);
        cudaFree(b.off);
        b.half = nullptr;
        b.off = nullptr;
    }
    const int64_t n = [&]() { int64_t v = 0; cudaMemcpy(&v, b.ptr + b.nrows, sizeof(int64_t), cudaMemcpyDeviceToHost); return v; }();
    p->device_bytes -= b.bytes;
    const size_t xt_len = b.order == 1   ? (size_t)((b.gh + 3) / 4) * ((b.gw + 3) / 4) * 16
                          : b.order == 4 ? (size_t)((b.gh + 7) / 8) * ((b.gw + 1) / 2) * 16
                          : b.order == 5 ? (size_t)((b.gh + 1) / 2) * ((b.gw + 7) / 8) * 16
                                         : (size_t)b.veclen;
    b.bytes = sizeof(int64_t) * (b.nrows + 1) +
              (keep_cmp ? sizeof(uint16_t) * (size_t)n + sizeof(int2) * (size_t)(n / (4 * b.gb)) : sizeof(int32_t) * (size_t)n) +
              sizeof(V) * (size_t)n + (b.xt ? sizeof(double) * xt_len : 0);
    p->device_bytes += b.bytes;
    return BSGD_OK;
}

static bool blocked_on(const bsgd_plan *p) {
    static const bool off = getenv("BSGD_NO_BLOCKED") != nullptr;
    return p->fb.ok && !off;
}
static bool blocked_tr_on(const bsgd_plan *p) { return p->tb.ok; }

template <typename V, class E>
static int launch_fwd(const bsgd_plan *p, const double *vec, const E &e, double *part, int64_t *cnt, cudaStream_t st) {
    if (p->stacked()) return launch_stacked_dir<V>(p, false, vec, e, part, cnt, st);
    if (gtiles_on(p->gf)) return launch_gtile<V>(p->gf, vec, e, part, cnt, st);
    if (blocked_on(p)) return launch_blocked<V>(p->fb, false, vec, e, part, cnt, st);
    return launch_one<V>(fwd_csr<V>(p, vec), p->g_fwd, e, part, cnt, p->nnz, st);
}

template <typename V, class E>
static int launch_tr(const bsgd_plan *p, const double *vec, const E &e, double *part, int64_t *cnt, cudaStream_t st) {
    if (p->stacked()) return launch_stacked_dir<V>(p, true, vec, e, part, cnt, st);
    if (blocked_tr_on(p)) return launch_blocked<V>(p->tb, true, vec, e, part, cnt, st);
    if (gtiles_on(p->gt)) return launch_gtile<V>(p->gt, vec, e, part, cnt, st);
    return launch_one<V>(tr_csr<V>(p, vec), p->g_tr, e, part, cnt, p->nnz, st);
}

#define DISPATCH_V(p, ...)                                          \
    ((p)->vdt == BSGD_F32 ? [&]() { using V = float; return __VA_ARGS__; }() \
                          : [&]() { using V = double; return __VA_ARGS__; }())

// ---------------------------------------------------------------------------
// workspace layout (shared by the epoch pieces and the standalone prox)
// ---------------------------------------------------------------------------
struct Ws {
    int64_t *ctl;    // [0] nx  [1] nr  [2] scratch count
    double *scal;    // prox scalars + reduction results
    double *xpart;   // [kMaxPartials * 4]
    double *rpart;   // [kMaxPartials]
    double *red;     // [2 * kMaxPartials * kPwMaxK]
    double *uimg;    // [cols]
    double *fields;  // [10 * n]: p, q, c for up to three axes, the split prox's u field
};

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

// Stride between the prox's dual fields, in doubles.  Fields read at the same
// voxel index in one pass (p, q, c per axis, u) must not sit a power of two
// apart: at 256^3 a field is exactly 128 MiB, and equal-offset addresses then
// collide in the L2 / HBM channel hashing -- the 3-D prox ran 12.2 ms or
// 16-29 ms depending on where the workspace landed.  An odd multiple of 256 B
// between fields breaks the alignment.
static int64_t field_stride(int64_t n) { return ((n + 31) & ~(int64_t)31) + 96; }

static size_t ws_layout(void *base, int64_t cols, int64_t hw, Ws *ws) {
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += a256(bytes); return (char *)base + o; };
    char *ctl = take(sizeof(int64_t) * 16);
    char *scal = take(sizeof(double) * 32);
    char *xpart = take(sizeof(double) * kMaxPartials * 4);
    char *rpart = take(sizeof(double) * kMaxPartials);
    char *red = take(sizeof(double) * 2 * kMaxPartials * kPwMaxK);
    (void)take(sizeof(double) * 96);  // keep uimg off the fields' alignment (see field_stride)
    char *uimg = take(sizeof(double) * (size_t)std::max<int64_t>(cols, 1));
    char *fields = take(sizeof(double) * kProxFields * (size_t)(hw > 0 ? field_stride(hw) : 0));
    if (ws) {
        ws->ctl = (int64_t *)ctl; ws->scal = (double *)scal; ws->xpart = (double *)xpart;
        ws->rpart = (double *)rpart; ws->red = (double *)red; ws->uimg = (double *)uimg;
        ws->fields = (double *)fields;
    }
    return off;
}

// ---------------------------------------------------------------------------
// small reduction kernels
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) dot_part_kernel(int64_t n, const double *a, const double *b, int mode,
                                                            double *part) {
    __shared__ double sm[kThreads / 32];
    double v[1] = {0.0};
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        if (mode == 0) v[0] += a[k] * b[k];
        else { const double d = a[k] - b[k]; v[0] += d * d; }
    }
    block_sum<1>(v, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void sum_parts_kernel(const double *part, int n, double *out) {
    double v[1];
    warp_sum_partials<1>(part, n, v);
    if (threadIdx.x == 0) out[0] = v[0];
}

__global__ void sum_counted_kernel(const double *part, const int64_t *cnt, double *out) {
    double v[1];
    warp_sum_partials<1>(part, (int)cnt[0], v);
    if (threadIdx.x == 0) out[0] = v[0];
}

__global__ void assemble_kernel(int64_t rows, int64_t N, const double *y, const double *z, double *out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        double acc = y[r];
        for (int64_t j = 0; j < N; ++j) acc = rn_sub(acc, z[j * rows + r]);
        out[r] = acc;
    }
}

__global__ void set_info_kernel(int32_t *info, int32_t a, int32_t b, int32_t c, int32_t d) {
    info[0] = a; info[1] = b; info[2] = c; info[3] = d;
}

struct TailArgs {
    const int64_t *ctl;
    const double *xpart;
    const double *rpart;
    const double *scal;
    const double *fnext_dev;
    int fnext_mode;  // 0 none, 1 from rpart, 2 from fnext_dev
    int monitor;
    int has_prox;
    double mu;
    double *f_curr;
    double *history;
    int64_t *counter;
    int64_t cap;
};

__global__ void tail_kernel(TailArgs t) {
    double xs[4];
    warp_sum_partials<4>(t.xpart, (int)t.ctl[0], xs);
    double fn = __longlong_as_double(0x7ff8000000000000LL);
    if (t.fnext_mode == 1) {
        double r[1];
        warp_sum_partials<1>(t.rpart, (int)t.ctl[1], r);
        fn = r[0];
    } else if (t.fnext_mode == 2) {
        fn = t.fnext_dev[0];
    }
    if (threadIdx.x == 0) {
        const int64_t row = t.counter[0];
        const double fc = t.f_curr != nullptr ? t.f_curr[0] : 0.0;
        double holds = -1.0;
        if (t.monitor) {
            // sufficient_decrease_holds (solvers.py:198-215): f_next < f_curr + d.(-g) + |d|^2/(2 mu)
            double bound = rn_add(fc, -xs[2]);
            bound = rn_add(bound, xs[3] / (2.0 * t.mu));
            holds = (fn < bound) ? 1.0 : 0.0;
            t.f_curr[0] = fn;
        }
        if (row >= 0 && row < t.cap) {
            double *h = t.history + row * BSGD_HIST_COLS;
            h[BSGD_H_FNEXT] = fn;
            h[BSGD_H_HOLDS] = holds;
            h[BSGD_H_XX] = xs[0];
            h[BSGD_H_XE] = xs[1];
            h[BSGD_H_TV] = t.has_prox ? t.scal[0] : 0.0;
            h[BSGD_H_PITER] = t.has_prox ? t.scal[1] : 0.0;
            h[BSGD_H_PRESTART] = t.has_prox ? t.scal[2] : 0.0;
            h[BSGD_H_PCONV] = t.has_prox ? t.scal[3] : 0.0;
            h[BSGD_H_PFELL] = t.has_prox ? t.scal[4] : 0.0;
            h[BSGD_H_DG] = xs[2];
            h[BSGD_H_DD] = xs[3];
            h[BSGD_H_FCURR] = fc;
        }
        t.counter[0] = row + 1;
    }
}

// ---------------------------------------------------------------------------
// prox launch
// ---------------------------------------------------------------------------
template <int DIM>
static size_t prox_dyn_smem() { return sizeof(double) * (1 + 2 * DIM) * fgp_chunk<DIM>() * 128; }

template <int DIM, bool FAST>
static int prox_occupancy() {
    static int occ = 0;
    if (occ == 0) {
        cudaFuncSetAttribute(fgp_kernel<DIM, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)prox_dyn_smem<DIM>());
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fgp_kernel<DIM, FAST>, kThreads, prox_dyn_smem<DIM>());
        if (occ < 1) occ = 1;
    }
    return occ;
}

// dynamic shared memory of the split / slab sum passes (pw_cta_fast chunks of 8 leaves)
// (the fast path sums leaves directly, pw_cta_direct: no dynamic buffer)
template <int K>
static size_t slab_smem(bool) { return 0; }

// Grid of the grid-stride stencil passes (candidate, finalize, output): exactly
// the CTAs that are resident at once, so the whole grid sweeps the volume
// together and a voxel's neighbour planes are still in L2 when it is reached.
// With 8 CTAs per SM requested but 5 resident (48 registers), the late CTAs
// re-swept the volume after the others and re-read their neighbour planes from
// DRAM (candidate pass: 851 MB read for 537 MB of fields, profiles/r01_c5.md).
template <int DIM>
static int stencil_grid(int64_t n) {
    static int occ = 0;
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slab_candidate_kernel<DIM>, kThreads, 0);
        if (occ < 1) occ = 1;
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, kThreads), (int64_t)num_sms() * occ));
}

template <int DIM>
static int cand_u_occupancy() {
    static int occ = 0;
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slab_cand_u_kernel<DIM, 4>, kThreads, 0);
        if (occ < 1) occ = 1;
    }
    return occ;
}

template <int DIM>
static void split_attrs() {
    static bool done = false;
    if (done) return;
    done = true;
    cudaFuncSetAttribute(slab_init_kernel<DIM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)slab_smem<2>(true));
    cudaFuncSetAttribute(slab_energy_kernel<DIM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)slab_smem<2>(true));
    cudaFuncSetAttribute(slab_dual_kernel<DIM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)slab_smem<1 + 2 * DIM>(true));
}

template <int DIM>
static void prox_warm() {
    (void)prox_occupancy<DIM, true>();
    (void)prox_occupancy<DIM, false>();
    split_attrs<DIM>();
    (void)cand_u_occupancy<DIM>();
}

// Split prox (slab.cuh): one kernel per FGP pass with the decisions on the
// device, for volumes whose fields do not stay in L2.  A fixed launch sequence
// (passes that do not apply return at once), so it is graph-capturable.
// BSGD_PROX_CANDIDATE=fused: the one-pass 3-D candidate (experiments / tests)
static int getenv_candidate_fused() {
    const char *e = getenv("BSGD_PROX_CANDIDATE");
    return (e && strcmp(e, "fused") == 0) ? 1 : 0;
}

template <int DIM>
static int launch_prox_split(const ProxArgs &a, cudaStream_t st) {
    split_attrs<DIM>();
    SlabView v = {};
    v.a = a;
    v.off = 0;
    v.n = a.N;
    v.ds = a.ds;
    v.fast = a.fast;
    const int64_t S = (int64_t)1 << a.ds;
    // CTAs of the sum passes: 32 leaves each (one 4-leaf group per warp), at most
    // 4096 (the partials buffer).  Fine grains balance the SMs: 256^3 with 512
    // CTAs (4 on 68 SMs, 3 on the rest) 5.45 ms for 10 iterations, 4096: 5.06 ms
    v.G = (int)std::max<int64_t>(1, std::min<int64_t>(S / 32, 4096));
    if (const char *e = getenv("BSGD_SPLIT_G")) {   // experiments: CTAs of the sum passes (power of two)
        const int g = atoi(e);
        if (g >= 1 && (g & (g - 1)) == 0 && g <= 4096) v.G = (int)std::min<int64_t>(S, g);
    }
    if (v.fast && S / v.G > kPwMaxQ) v.fast = 0;   // direct leaf sums hold <= kPwMaxQ leaves per CTA
    if (S / v.G > kPwMaxQ * (int64_t)(v.fast ? 1 : kThreads / 8))
        return fail(BSGD_EINVAL, "image too large for the pairwise tree (%lld voxels)", (long long)a.N);
    v.ctl = (FgpCtl *)(a.red + (size_t)kMaxPartials * kPwMaxK);
    // the control block shares the reduction buffer with the other prox kernels:
    // clear it (the folded decisions count arriving CTAs in it)
    CU(cudaMemsetAsync(v.ctl, 0, sizeof(FgpCtl), st));
    double *part = a.red;
    // p = q = 0 (tv.py:198-201): the first iteration's passes read them as literal
    // zeros (v.zero) and write every voxel of c and q, so nothing is cleared; only
    // a prox without iterations needs the stored zeros (for the finalize pass)
    if (a.max_iters < 1)
        for (int k = 0; k < DIM; ++k) {
            CU(cudaMemsetAsync(a.f[k], 0, sizeof(double) * a.N, st));
            CU(cudaMemsetAsync(a.f[DIM + k], 0, sizeof(double) * a.N, st));
        }
    const int grid = stencil_grid<DIM>(a.N);
    constexpr int KD = 1 + 2 * DIM;
    const bool fast = v.fast != 0;
    auto sums2 = [&](bool energy) {
        if (energy) {
            if (fast) slab_energy_kernel<DIM, true><<<v.G, kThreads, slab_smem<2>(true), st>>>(v, part);
            else slab_energy_kernel<DIM, false><<<v.G, kThreads, 0, st>>>(v, part);
        } else {
            if (fast) slab_init_kernel<DIM, true><<<v.G, kThreads, slab_smem<2>(true), st>>>(v, part);
            else slab_init_kernel<DIM, false><<<v.G, kThreads, 0, st>>>(v, part);
        }
    };
    // volumes: the candidate reads a stored u field (f[kProxFields - 1]) instead of
    // evaluating u = b + w div src four times per voxel (256^3: 0.55-0.65 ms fused,
    // issue-bound), and the dual pass writes the next iteration's u' from q' in
    // the same sweep, so an iteration is two passes (the first candidate reads b;
    // a restart takes the one-pass candidate from p)
    const bool two_pass = DIM == 3 && getenv_candidate_fused() == 0;
    double *ufield = a.f[kProxFields - 1];
    auto dual = [&]() {
        if (two_pass) {
            if (fast) slab_dual_u_kernel<DIM, true><<<v.G, kThreads, slab_smem<KD>(true), st>>>(v, part, ufield);
            else slab_dual_u_kernel<DIM, false><<<v.G, kThreads, 0, st>>>(v, part, ufield);
        } else {
            if (fast) slab_dual_kernel<DIM, true><<<v.G, kThreads, slab_smem<KD>(true), st>>>(v, 0.0, part);
            else slab_dual_kernel<DIM, false><<<v.G, kThreads, 0, st>>>(v, 0.0, part);
        }
    };
    // every sum pass takes its own decision in its last CTA (slab_fold_decide):
    // per FGP iteration 2 launches on the main path and 2 (returning at once
    // unless a restart was decided) on the restart path
    v.when = 0;
    v.fold_stage = 0;
    v.fold_it = 0;
    sums2(false);
    auto candidate = [&](int from_p) {
        if (two_pass && !from_p) {
            // 4 CTAs per SM (64 registers, no spill), the grid = the CTAs resident at
            // once (one sweep; 3 per SM at 71 registers with a 4-per-SM grid swept twice:
            // 6.3 vs 5.4 ms for the 256^3 prox; 5 / 6 per SM spill and measured no better)
            const int grid_cu = (int)std::max<int64_t>(
                1, std::min<int64_t>(cdiv(v.n, kThreads), (int64_t)num_sms() * cand_u_occupancy<DIM>()));
            slab_cand_u_kernel<DIM, 4><<<grid_cu, kThreads, 0, st>>>(v, 0, ufield);
        } else {   // restarts (rare) take the one-pass candidate from p
            slab_candidate_kernel<DIM><<<grid, kThreads, 0, st>>>(v, from_p);
        }
    };
    for (int it = 0; it < a.max_iters; ++it) {
        v.zero = it == 0 ? 1 : 0;
        v.fold_it = it;
        v.when = 1;  // unless converged
        v.fold_stage = -1;
        candidate(0);            // u' of the last accepted dual pass (b itself at it = 0)
        v.fold_stage = 1;
        dual();
        v.when = 2;  // only on a restart
        v.fold_stage = -1;
        candidate(1);
        v.fold_stage = 2;
        dual();
    }
    v.when = 0;
    v.zero = 0;
    v.fold_stage = -1;
    slab_finalize_kernel<DIM><<<grid, kThreads, 0, st>>>(v);
    v.fold_stage = 3;
    sums2(true);
    v.fold_stage = -1;
    split_output_kernel<DIM><<<grid, kThreads, 0, st>>>(v);
    LAUNCHED();
    return BSGD_OK;
}

static bool prox_split_on(const ProxArgs &a) {
    const char *e = getenv("BSGD_PROX_SPLIT");
    if (e && e[0]) return e[0] == '1';
    return a.N >= ((int64_t)1 << 21);
}

template <int DIM, bool FAST>
static int launch_prox_dim(ProxArgs &a, cudaStream_t st) {
    const int occ = prox_occupancy<DIM, FAST>();
    // G: a power of two (numpy-order top tree), co-resident, <= 512
    int grid = pow2_floor(std::max<int64_t>(1, std::min<int64_t>((int64_t)occ * num_sms(), 512)));
    const int64_t S = (int64_t)1 << a.ds;
    const int64_t per_slot = FAST ? fgp_chunk<DIM>() : kThreads / 8;  // subtrees folded per smem slot
    if (S / grid > kPwMaxQ * per_slot)
        return fail(BSGD_EINVAL, "image too large for the pairwise tree (%lld pixels)", (long long)a.N);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = prox_dyn_smem<DIM>();
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelEx(&cfg, fgp_kernel<DIM, FAST>, a));
    return BSGD_OK;
}

// a.D <= 1: 2D image (tv.py); a.D >= 2: 3D volume (oracle tv_prox3)
static int launch_prox(ProxArgs &a, cudaStream_t st) {
    int rc = pw_depth(a.N, &a.ds);
    if (rc) return rc;
    a.fast = (a.N % 128 == 0 && a.N / 128 == ((int64_t)1 << a.ds)) ? 1 : 0;
    const bool split = prox_split_on(a);
    if (a.D <= 1) {
        a.D = 1;
        if (split) return launch_prox_split<2>(a, st);
        // power-of-two images up to 1024 wide: the row-walk kernel (one grid barrier per
        // FGP iteration, fgp2.cu); BSGD_PROX_KERNEL=coop selects fgp_kernel (tests compare them)
        const char *pk = getenv("BSGD_PROX_KERNEL");
        if (!(pk && strcmp(pk, "coop") == 0) && fgp2_rows_supported(a)) {
            cudaError_t e = fgp2_rows_launch(a, num_sms(), st);
            if (e == cudaSuccess) return BSGD_OK;
            if (e != cudaErrorCooperativeLaunchTooLarge) return fail(BSGD_ECUDA, "fgp2_rows_kernel: %s", cudaGetErrorString(e));
            cudaGetLastError();
        }
        return a.fast ? launch_prox_dim<2, true>(a, st) : launch_prox_dim<2, false>(a, st);
    }
    if (split) return launch_prox_split<3>(a, st);
    return a.fast ? launch_prox_dim<3, true>(a, st) : launch_prox_dim<3, false>(a, st);
}

static void prox_fields(ProxArgs &a, const Ws &ws, int64_t n) {
    for (int k = 0; k < kProxFields; ++k) a.f[k] = ws.fields + (size_t)k * field_stride(n);
    a.red = ws.red;
}

// Build the tile-staged copy of A2 (transposed = 0) or A2^T (1) from a host row
// grouping: tile t holds stored rows tile_rows[tile_ptr[t] .. tile_ptr[t+1]).
template <typename V>
static int build_stk_tiles(bsgd_plan *p, bool tr, int64_t ntiles, const int64_t *tptr, const int64_t *trows,
                           cudaStream_t st) {
    const int64_t nrows = tr ? p->scols : p->srows, nnz = p->snnz;
    if (tptr[0] != 0) return fail(BSGD_EINVAL, "tile_ptr must start at 0");
    if ((tr ? p->srows : p->scols) >= ((int64_t)1 << 24))
        return fail(BSGD_EINVAL, "tile-staged products need fewer than 2^24 stored columns");
    const int64_t ntr = tptr[ntiles];
    if (ntr != nrows) return fail(BSGD_EINVAL, "tiles must cover every stored row exactly once (%lld of %lld)",
                                  (long long)ntr, (long long)nrows);
    std::vector<char> seen(nrows, 0);
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t n = tptr[t + 1] - tptr[t];
        if (n < 1 || n > kTileRows) return fail(BSGD_EINVAL, "tile %lld has %lld rows (1..%d)", (long long)t, (long long)n, kTileRows);
    }
    for (int64_t i = 0; i < ntr; ++i) {
        const int64_t r = trows[i];
        if (r < 0 || r >= nrows || seen[r]) return fail(BSGD_EINVAL, "tile rows must be a permutation of the stored rows");
        seen[r] = 1;
    }
    std::vector<int64_t> ptr(nrows + 1);
    std::vector<int32_t> idx(nnz);
    std::vector<V> val(nnz);
    CU(cudaMemcpyAsync(ptr.data(), tr ? p->t_ptr : p->f_ptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(idx.data(), tr ? p->t_idx : p->f_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(val.data(), tr ? p->t_val : p->f_val, sizeof(V) * nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    // Eight slices per consumer lane for A's rows (rays) when the depth allows (a
    // multiple of 256: the entry decode serves twice the slices), with half as
    // many columns per segment so a stage's window stays 32 KB.  configs[4]: A
    // 2.86 -> 2.62 ms; A^T (pixel rows) ran 3.21 -> 5.09 ms that way and keeps
    // four.  BSGD_STK_KZ=4 / 8 forces either for both.
    int kz = (!tr && p->depth % 256 == 0) ? 8 : 4;
    if (const char *e = getenv("BSGD_STK_KZ")) kz = atoi(e) == 8 && p->depth % 256 == 0 ? 8 : 4;
    const int64_t seg = kz == 8 ? tile_seg<8>() : tile_seg<4>();
    // per tile: sorted distinct columns, cut into segments of seg columns; per segment
    // the tile rows' entries inside it (row-major, position in the segment as uint8)
    struct TileOut {
        std::vector<int32_t> uni;
        std::vector<int32_t> nj;
        std::vector<std::array<uint16_t, 24>> rows;
        std::vector<uint8_t> loc;   // per segment, padded to 16
        std::vector<V> val;
        std::vector<int32_t> col;
        std::vector<int64_t> ent;   // per segment entry offset inside this tile's arrays
    };
    std::vector<TileOut> outs(ntiles);
    unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nth; ++w) {
        pool.emplace_back([&, w]() {
            std::vector<int32_t> cols;
            for (int64_t t = w; t < ntiles; t += nth) {
                TileOut &o = outs[t];
                cols.clear();
                for (int64_t i = tptr[t]; i < tptr[t + 1]; ++i) {
                    const int64_t r = trows[i];
                    cols.insert(cols.end(), idx.begin() + ptr[r], idx.begin() + ptr[r + 1]);
                }
                std::sort(cols.begin(), cols.end());
                cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
                o.uni = cols;
                const int64_t nu = (int64_t)cols.size();
                const int64_t nseg = std::max<int64_t>(1, (nu + seg - 1) / seg);
                const int64_t nrt = tptr[t + 1] - tptr[t];
                std::vector<int64_t> cur(nrt);
                for (int64_t i = 0; i < nrt; ++i) cur[i] = ptr[trows[tptr[t] + i]];
                for (int64_t sg = 0; sg < nseg; ++sg) {
                    const int64_t j0 = sg * seg, j1 = std::min<int64_t>(nu, j0 + seg);
                    const int32_t cmax = j1 > j0 ? cols[j1 - 1] : -1;
                    std::array<uint16_t, 24> ro{};
                    o.ent.push_back((int64_t)o.loc.size());
                    int n = 0;
                    for (int64_t i = 0; i < nrt; ++i) {
                        const int64_t r = trows[tptr[t] + i];
                        ro[i] = (uint16_t)n;
                        while (cur[i] < ptr[r + 1] && idx[cur[i]] <= cmax) {
                            const int64_t pos = std::lower_bound(cols.begin() + j0, cols.begin() + j1, idx[cur[i]]) - cols.begin();
                            o.loc.push_back((uint8_t)(pos - j0));
                            o.val.push_back(val[cur[i]]);
                            o.col.push_back(idx[cur[i]]);
                            ++cur[i];
                            ++n;
                        }
                    }
                    for (int64_t i = nrt; i <= kTileRows; ++i) ro[i] = (uint16_t)n;
                    while (o.loc.size() % 16) { o.loc.push_back(0); o.val.push_back((V)0); o.col.push_back(0); }
                    o.rows.push_back(ro);
                    o.nj.push_back((int32_t)(j1 - j0));
                }
            }
        });
    }
    for (auto &th : pool) th.join();
    // flatten: segment g's column ids at uni[g * seg ..] (zero padded)
    int64_t nseg_all = 0, nent = 0;
    std::vector<int64_t> seg_ptr(ntiles + 1, 0);
    for (int64_t t = 0; t < ntiles; ++t) {
        seg_ptr[t + 1] = seg_ptr[t] + (int64_t)outs[t].nj.size();
        nent += (int64_t)outs[t].loc.size();
    }
    nseg_all = seg_ptr[ntiles];
    std::vector<int64_t> seg_uni(nseg_all), seg_ent(nseg_all);
    std::vector<int32_t> seg_nj(nseg_all), uni((size_t)std::max<int64_t>(nseg_all, 1) * seg, 0);
    std::vector<uint16_t> seg_row((size_t)nseg_all * 24);
    std::vector<TileEnt<V>> ents(std::max<int64_t>(nent, 16));
    int64_t eo = 0;
    for (int64_t t = 0; t < ntiles; ++t) {
        const TileOut &o = outs[t];
        int64_t src = 0;
        for (size_t sg = 0; sg < o.nj.size(); ++sg) {
            const int64_t g = seg_ptr[t] + (int64_t)sg;
            const int32_t nj = o.nj[sg];
            seg_uni[g] = g * seg;
            seg_nj[g] = nj;
            seg_ent[g] = eo + o.ent[sg];
            std::copy(o.rows[sg].begin(), o.rows[sg].end(), seg_row.begin() + g * 24);
            std::copy(o.uni.begin() + src, o.uni.begin() + src + nj, uni.begin() + g * seg);
            src += nj;
        }
        for (size_t q = 0; q < o.loc.size(); ++q) {
            ents[eo + q].val = o.val[q];
            ents[eo + q].cl = (uint32_t)o.col[q] << 8 | o.loc[q];
        }
        eo += (int64_t)o.loc.size();
    }
    std::vector<int32_t> trows32(ntr);
    for (int64_t i = 0; i < ntr; ++i) trows32[i] = (int32_t)trows[i];
    bsgd_plan::StkTileStore &S = tr ? p->stt : p->sf;
    stk_tiles_free(S);
    bsgd_plan::StkTileStore N;
    auto up = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(bytes, 16));
        if (e == cudaSuccess) e = cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st);
        N.bytes += bytes;
        return e;
    };
    cudaError_t e = up((void **)&N.tile_ptr, tptr, sizeof(int64_t) * (ntiles + 1));
    if (e == cudaSuccess) e = up((void **)&N.tile_rows, trows32.data(), sizeof(int32_t) * ntr);
    if (e == cudaSuccess) e = up((void **)&N.seg_ptr, seg_ptr.data(), sizeof(int64_t) * (ntiles + 1));
    if (e == cudaSuccess) e = up((void **)&N.seg_uni, seg_uni.data(), sizeof(int64_t) * nseg_all);
    if (e == cudaSuccess) e = up((void **)&N.seg_nj, seg_nj.data(), sizeof(int32_t) * nseg_all);
    if (e == cudaSuccess) e = up((void **)&N.seg_ent, seg_ent.data(), sizeof(int64_t) * nseg_all);
    if (e == cudaSuccess) e = up((void **)&N.seg_row, seg_row.data(), sizeof(uint16_t) * seg_row.size());
    if (e == cudaSuccess) e = up((void **)&N.uni, uni.data(), sizeof(int32_t) * uni.size());
    if (e == cudaSuccess) e = up(&N.ent, ents.data(), sizeof(TileEnt<V>) * ents.size());
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        stk_tiles_free(N);
        return fail(e == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA, "tile upload failed: %s",
                    cudaGetErrorString(e));
    }
    N.ntiles = ntiles;
    N.kz = kz;
    N.ok = true;
    S = N;
    p->device_bytes += N.bytes;
    return BSGD_OK;
}

// Build the gather-tiled copy of A (transposed = 0) or A^T (1) of an ordinary
// plan from a host row grouping (tile t = rows tile_rows[tile_ptr[t] ..]).
template <typename V>
static int build_gtiles(bsgd_plan *p, bool tr, int64_t ntiles, const int64_t *tptr, const int64_t *trows,
                        cudaStream_t st) {
    const int64_t nrows = tr ? p->cols : p->rows, nnz = p->nnz;
    if (tptr[0] != 0 || tptr[ntiles] != nrows)
        return fail(BSGD_EINVAL, "tiles must cover every row exactly once");
    std::vector<char> seen(nrows, 0);
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t n = tptr[t + 1] - tptr[t];
        if (n < 1 || n > kGTileRows) return fail(BSGD_EINVAL, "tile %lld has %lld rows (1..%d)", (long long)t, (long long)n, kGTileRows);
    }
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t r = trows[i];
        if (r < 0 || r >= nrows || seen[r]) return fail(BSGD_EINVAL, "tile rows must be a permutation of the rows");
        seen[r] = 1;
    }
    std::vector<int64_t> ptr(nrows + 1);
    std::vector<int32_t> idx(nnz);
    std::vector<V> val(nnz);
    CU(cudaMemcpyAsync(ptr.data(), tr ? p->t_ptr : p->f_ptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(idx.data(), tr ? p->t_idx : p->f_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(val.data(), tr ? p->t_val : p->f_val, sizeof(V) * nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    // rows padded to whole stream blocks (gtile.cuh: entry e = 16 m + l of a block at 8 l + m)
    std::vector<int64_t> rptr(nrows + 1, 0);
    for (int64_t i = 0; i < nrows; ++i) {
        const int64_t r = trows[i];
        const int64_t len = ptr[r + 1] - ptr[r];
        rptr[i + 1] = rptr[i] + (len + kGTileBlock - 1) / kGTileBlock * kGTileBlock;
    }
    const int64_t nstore = rptr[nrows];
    auto slot = [](int64_t k) { const int64_t e = k % kGTileBlock; return k - e + (e % 16) * 8 + e / 16; };
    std::vector<uint16_t> loc(std::max<int64_t>(nstore, 1), 0);
    std::vector<V> pval(std::max<int64_t>(nstore, 1), V(0));
    std::vector<std::vector<int32_t>> unions(ntiles);
    unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    std::vector<int> big(nth, 0);
    for (unsigned w = 0; w < nth; ++w) {
        pool.emplace_back([&, w]() {
            std::vector<int32_t> cols;
            for (int64_t t = w; t < ntiles; t += nth) {
                cols.clear();
                for (int64_t i = tptr[t]; i < tptr[t + 1]; ++i) {
                    const int64_t r = trows[i];
                    cols.insert(cols.end(), idx.begin() + ptr[r], idx.begin() + ptr[r + 1]);
                }
                std::sort(cols.begin(), cols.end());
                cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
                if (cols.size() > 28000) { big[w] = 1; continue; }
                for (int64_t i = tptr[t]; i < tptr[t + 1]; ++i) {
                    const int64_t r = trows[i];
                    for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
                        const int64_t o = rptr[i] + slot(k - ptr[r]);
                        loc[o] = (uint16_t)(std::lower_bound(cols.begin(), cols.end(), idx[k]) - cols.begin());
                        pval[o] = val[k];
                    }
                }
                unions[t] = cols;
            }
        });
    }
    for (auto &th : pool) th.join();
    for (int b : big)
        if (b) return fail(BSGD_EINVAL, "a tile's rows touch more than 28000 distinct columns");
    std::vector<int64_t> uptr(ntiles + 1, 0);
    int max_union = 0;
    for (int64_t t = 0; t < ntiles; ++t) {
        uptr[t + 1] = uptr[t] + (int64_t)unions[t].size();
        max_union = std::max(max_union, (int)unions[t].size());
    }
    std::vector<int32_t> uni(std::max<int64_t>(uptr[ntiles], 1));
    for (int64_t t = 0; t < ntiles; ++t) std::copy(unions[t].begin(), unions[t].end(), uni.begin() + uptr[t]);
    std::vector<int32_t> trows32(nrows);
    for (int64_t i = 0; i < nrows; ++i) trows32[i] = (int32_t)trows[i];
    bsgd_plan::GTileStore &S = tr ? p->gt : p->gf;
    p->device_bytes -= S.bytes;
    gtiles_free(S);
    bsgd_plan::GTileStore N;
    auto up = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(bytes, 16));
        if (e == cudaSuccess) e = cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st);
        N.bytes += bytes;
        return e;
    };
    cudaError_t e = up((void **)&N.tile_ptr, tptr, sizeof(int64_t) * (ntiles + 1));
    if (e == cudaSuccess) e = up((void **)&N.tile_rows, trows32.data(), sizeof(int32_t) * nrows);
    if (e == cudaSuccess) e = up((void **)&N.row_ptr, rptr.data(), sizeof(int64_t) * (nrows + 1));
    if (e == cudaSuccess) e = up((void **)&N.loc, loc.data(), sizeof(uint16_t) * nstore);
    if (e == cudaSuccess) e = up(&N.val, pval.data(), sizeof(V) * nstore);
    if (e == cudaSuccess) e = up((void **)&N.uni_ptr, uptr.data(), sizeof(int64_t) * (ntiles + 1));
    if (e == cudaSuccess) e = up((void **)&N.uni, uni.data(), sizeof(int32_t) * uni.size());
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        gtiles_free(N);
        return fail(e == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA, "tile upload failed: %s",
                    cudaGetErrorString(e));
    }
    N.ntiles = ntiles;
    N.max_union = max_union;
    N.ok = true;
    S = N;
    p->device_bytes += N.bytes;
    return BSGD_OK;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// slab-decomposed prox (multi-GPU): workspace layout and launch helpers
// ---------------------------------------------------------------------------
constexpr int kSlabPartials = 8192;   // doubles: G <= 512 CTAs x K <= 7 sums, or G x 4 stats
constexpr int kSlabCtlOffset = 32;     // FgpCtl of the device-decided slab prox, after the sums (16) and stats
static_assert(sizeof(FgpCtl) <= 96 * sizeof(double), "control block must fit the slot's padding");

static int64_t slab_halo(int64_t depth, int64_t height, int64_t width) {
    return depth > 1 ? height * width : width;
}

// offsets in doubles; returns the total size in doubles
static int64_t slab_offsets(int64_t depth, int64_t height, int64_t width, int64_t count, int64_t *off) {
    const int dim = depth > 1 ? 3 : 2;
    const int64_t len = count + 2 * slab_halo(depth, height, width);
    const int64_t stride = field_stride(len);
    int64_t o = kSlabPartials + 32;   // partials, then the sums slot (16) and stats (16)
    off[11] = kSlabPartials;
    o += 96;
    off[0] = o; o += stride;
    for (int grp = 0; grp < 3; ++grp)
        for (int k = 0; k < 3; ++k) {
            if (k < dim) { off[1 + 3 * grp + k] = o; o += stride; }
            else off[1 + 3 * grp + k] = -1;
        }
    off[10] = o; o += stride;
    return o;
}

struct SlabCtx {
    SlabView v;
    double *part;
    double *stats;
    int dim;
    int G;        // CTAs of the sum passes (power of two)
    int grid;     // CTAs of the elementwise passes
};

static int slab_ctx(const bsgd_slab *s, SlabCtx &c, bool need_weight = true) {
    if (!s) return fail(BSGD_EINVAL, "slab is NULL");
    const int64_t D = s->depth < 1 ? 1 : s->depth;
    if (s->height < 1 || s->width < 1) return fail(BSGD_EINVAL, "slab dimensions must be positive");
    const int64_t N = D * s->height * s->width;
    if (N >= ((int64_t)1 << 31)) return fail(BSGD_EINVAL, "volume too large (%lld voxels)", (long long)N);
    if (s->offset < 0 || s->count < 1 || s->offset + s->count > N)
        return fail(BSGD_EINVAL, "slab [%lld, +%lld) outside the volume", (long long)s->offset, (long long)s->count);
    if (need_weight && !(s->weight > 0.0)) return fail(BSGD_EINVAL, "slab prox weight must be positive");
    if (s->parity != 0 && s->parity != 1) return fail(BSGD_EINVAL, "parity must be 0 or 1");
    int64_t off[BSGD_SLAB_SLOTS];
    const int64_t total = slab_offsets(D, s->height, s->width, s->count, off);
    if (!s->workspace || s->workspace_bytes < (size_t)total * sizeof(double))
        return fail(BSGD_EINVAL, "slab workspace too small");
    double *base = (double *)s->workspace;
    const int64_t h = slab_halo(D, s->height, s->width);
    // shifted so that ptr[p] addresses global voxel p (valid for p in [offset - h, offset + count + h))
    auto at = [&](int slot) { return base + off[slot] + h - s->offset; };
    c.dim = D > 1 ? 3 : 2;
    ProxArgs &a = c.v.a;
    a = ProxArgs{};
    a.D = D; a.H = s->height; a.W = s->width; a.N = N;
    a.b = at(0);
    a.w = s->weight;
    a.step = 1.0 / ((D > 1 ? 12.0 : 8.0) * s->weight);
    for (int k = 0; k < c.dim; ++k) {  // dual buffer 0, q, dual buffer 1 (slab_roles resolves p / c)
        a.f[k] = at(1 + k);
        a.f[c.dim + k] = at(7 + k);
        a.f[2 * c.dim + k] = at(4 + k);
    }
    c.v.parity = s->parity;
    c.v.when = 0;
    c.v.ctl = nullptr;
    c.v.zero = 0;
    if (s->flags & BSGD_SLAB_DEVICE) {   // decisions in the workspace's control block
        c.v.ctl = (FgpCtl *)(base + off[11] + kSlabCtlOffset);
        c.v.when = (s->flags >> 1) & 3;
    }
    c.v.ilv = 0;
    c.v.ilv_z0 = 0;
    c.v.fold_stage = -1;
    if (s->flags & BSGD_SLAB_INTERLEAVED) {   // solver vectors: this rank's slices, interleaved
        const int64_t hw = s->height * s->width;
        if (D <= 1 || s->offset % hw || s->count % hw)
            return fail(BSGD_EINVAL, "BSGD_SLAB_INTERLEAVED needs a volume slab of whole slices");
        c.v.ilv = s->count / hw;
        c.v.ilv_z0 = s->offset / hw;
    }
    c.v.u = at(10);
    c.v.off = s->offset;
    c.v.n = s->count;
    int rc = pw_depth(s->count, &c.v.ds);
    if (rc) return rc;
    c.v.fast = (s->count % 128 == 0 && s->count / 128 == ((int64_t)1 << c.v.ds)) ? 1 : 0;
    const int64_t S = (int64_t)1 << c.v.ds;
    c.G = (int)std::min<int64_t>(S, 512);
    c.v.G = c.G;
    if (c.v.fast && S / c.G > kPwMaxQ) c.v.fast = 0;   // direct leaf sums hold <= kPwMaxQ leaves per CTA
    const int64_t per_slot = c.v.fast ? 1 : kThreads / 8;
    if (S / c.G > kPwMaxQ * per_slot) return fail(BSGD_EINVAL, "slab too large for the pairwise tree");
    c.part = base;
    c.stats = base + off[11] + 16;
    c.grid = c.dim == 3 ? stencil_grid<3>(s->count) : stencil_grid<2>(s->count);
    return BSGD_OK;
}

template <int K, class Kern>
static int slab_sum_launch(const SlabCtx &c, Kern kern, size_t smem, double *out, cudaStream_t st) {
    if (smem > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<c.G, kThreads, smem, st>>>(c.v, c.part);
    slab_top_kernel<K><<<1, kThreads, 0, st>>>(c.v.ds, c.G, c.part, out);
    LAUNCHED();
    return BSGD_OK;
}

extern "C" {

const char *bsgd_last_error(void) { return g_err.c_str(); }

int bsgd_version(void) { return BSGD_VERSION; }

int bsgd_device_count(int *out) {
    if (!out) return fail(BSGD_EINVAL, "out is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) { cudaGetLastError(); n = 0; }
    *out = n;
    return BSGD_OK;
}

// everything after A's CSR is on the device: validation, A^T, tiled copies, block table
static int plan_finish(bsgd_plan *p, cudaStream_t st) {
    // stored CSR sizes (A2 for stacked plans)
    const int64_t rows = p->srows, cols = p->scols, nnz = p->snnz;
    const int value_dtype = p->vdt;
    const int64_t num_row_blocks = p->M, num_col_blocks = p->N;
    int rc = BSGD_OK;
#define PTRY(call)                                                                         \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            return fail(e_ == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA,        \
                        "%s failed: %s", #call, cudaGetErrorString(e_));                   \
        }                                                                                  \
    } while (0)
    const size_t vb = (size_t)value_dtype;
    PTRY(cudaMalloc(&p->t_ptr, sizeof(int64_t) * (cols + 1)));
    PTRY(cudaMalloc(&p->t_idx, sizeof(int32_t) * nnz));
    PTRY(cudaMalloc(&p->t_val, vb * nnz));
    PTRY(cudaMalloc(&p->d_row_bounds, sizeof(int64_t) * (num_row_blocks + 1)));
    PTRY(cudaMalloc(&p->d_col_bounds, sizeof(int64_t) * (num_col_blocks + 1)));
    p->device_bytes = sizeof(int64_t) * (rows + cols + 2) + 2 * (sizeof(int32_t) + vb) * nnz;
    PTRY(cudaMemcpyAsync(p->d_row_bounds, p->row_bounds.data(), sizeof(int64_t) * (num_row_blocks + 1),
                         cudaMemcpyHostToDevice, st));
    PTRY(cudaMemcpyAsync(p->d_col_bounds, p->col_bounds.data(), sizeof(int64_t) * (num_col_blocks + 1),
                         cudaMemcpyHostToDevice, st));
    if (p->stacked()) {  // block bounds in stored-index units when every bound is a multiple of depth
        auto upload = [&](const std::vector<int64_t> &b, int64_t **dst) -> int {
            for (int64_t v : b)
                if (v % p->depth) return BSGD_OK;
            std::vector<int64_t> q(b.size());
            for (size_t i = 0; i < b.size(); ++i) q[i] = b[i] / p->depth;
            PTRY(cudaMalloc(dst, sizeof(int64_t) * q.size()));
            PTRY(cudaMemcpy(*dst, q.data(), sizeof(int64_t) * q.size(), cudaMemcpyHostToDevice));
            return BSGD_OK;
        };
        rc = upload(p->col_bounds, &p->d_col_sbounds);
        if (!rc) rc = upload(p->row_bounds, &p->d_row_sbounds);
        if (rc) return rc;
    }
    // structural check (canonical form: sorted unique in-range indices per row)
    int *d_bad = nullptr;
    PTRY(cudaMalloc(&d_bad, sizeof(int)));
    PTRY(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    check_csr_kernel<<<grid_1d(rows), kThreads, 0, st>>>(rows, cols, p->f_ptr, p->f_idx, d_bad);
    int bad = 0;
    PTRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    PTRY(cudaStreamSynchronize(st));
    cudaFree(d_bad);
    if (bad) {
        return fail(BSGD_EINVAL, "CSR is not canonical (code %d: 1=indptr, 2=index range, 4=unsorted/duplicate)", bad);
    }
    rc = (value_dtype == BSGD_F32) ? build_transpose<float>(p, st) : build_transpose<double>(p, st);
    if (rc != BSGD_OK) return rc;
    rc = (value_dtype == BSGD_F32) ? build_blocked<float>(p, st) : build_blocked<double>(p, st);
    if (rc != BSGD_OK) return rc;
    rc = (value_dtype == BSGD_F32) ? tune_blocked<float>(p, p->fb) : tune_blocked<double>(p, p->fb);
    if (rc != BSGD_OK) return rc;
    // A^T's rows long too (a CT system handed over as a plain CSR: ~1.3 nonzeros per
    // angle and pixel): a blocked copy of A^T, gathered in tiles of the row grid when
    // infer_grid finds one (a sinogram), else in A^T's own column order;
    // bsgd_plan_blocked_transposed replaces it when the caller names the grid
    if (!p->stacked() && cols > 0 && (double)p->nnz / (double)cols >= 384.0 && !getenv("BSGD_NO_BLOCKED")) {
        int gh = 0, gw = 0;
        if (!infer_grid(p, true, st, &gh, &gw)) gh = gw = 0;
        rc = (value_dtype == BSGD_F32) ? build_blocked_dir<float>(p, true, gh, gw, st)
                                       : build_blocked_dir<double>(p, true, gh, gw, st);
        if (rc != BSGD_OK) return rc;
        rc = (value_dtype == BSGD_F32) ? tune_blocked<float>(p, p->tb) : tune_blocked<double>(p, p->tb);
        if (rc != BSGD_OK) return rc;
    }
    // block nnz table (blockops.py:179-180)
    unsigned long long *d_cnt = nullptr;
    const int64_t nb = num_row_blocks * num_col_blocks;
    PTRY(cudaMalloc(&d_cnt, sizeof(unsigned long long) * nb));
    PTRY(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * nb, st));
    if (p->stacked())
        stacked_block_nnz_kernel<<<grid_1d(p->rows), kThreads, 0, st>>>(p->f_ptr, p->f_idx, p->depth, p->rows,
                                                                        p->d_row_bounds, num_row_blocks,
                                                                        p->d_col_bounds, num_col_blocks, d_cnt);
    else
        block_nnz_kernel<<<grid_1d(rows), kThreads, 0, st>>>(rows, p->f_ptr, p->f_idx, num_row_blocks,
                                                             p->d_row_bounds, num_col_blocks, p->d_col_bounds, d_cnt);
    std::vector<unsigned long long> cnt(nb);
    PTRY(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned long long) * nb, cudaMemcpyDeviceToHost, st));
    PTRY(cudaStreamSynchronize(st));
    cudaFree(d_cnt);
    p->block_nnz.assign(cnt.begin(), cnt.end());
#undef PTRY
    // warm occupancy caches outside any graph capture
    prox_warm<2>();
    prox_warm<3>();
    return BSGD_OK;
}

static int plan_args_check(int64_t rows, int64_t cols, int64_t nnz, int value_dtype, int64_t num_row_blocks,
                           int64_t num_col_blocks, const int64_t *row_bounds, const int64_t *col_bounds, int device) {
    if (rows < 1 || cols < 1) return fail(BSGD_EINVAL, "matrix dimensions must be positive");
    if (cols >= ((int64_t)1 << 31) || rows >= ((int64_t)1 << 31))
        return fail(BSGD_EINVAL, "dimensions must be < 2^31 (int32 indices)");
    if (nnz == 0) return fail(BSGD_EINVAL, "matrix has no nonzeros");
    if (nnz < 0 || nnz >= ((int64_t)1 << 32)) return fail(BSGD_EINVAL, "nnz %lld out of range", (long long)nnz);
    if (value_dtype != BSGD_F32 && value_dtype != BSGD_F64) return fail(BSGD_EINVAL, "value dtype must be 4 or 8");
    if (!row_bounds || !col_bounds) return fail(BSGD_EINVAL, "NULL partition bounds");
    if (num_row_blocks < 1 || num_row_blocks > rows) return fail(BSGD_EINVAL, "row block count not in [1, rows]");
    if (num_col_blocks < 1 || num_col_blocks > cols) return fail(BSGD_EINVAL, "col block count not in [1, cols]");
    for (int64_t i = 0; i < num_row_blocks; ++i)
        if (row_bounds[i + 1] <= row_bounds[i]) return fail(BSGD_EINVAL, "row ranges must be nonempty and ascending");
    for (int64_t j = 0; j < num_col_blocks; ++j)
        if (col_bounds[j + 1] <= col_bounds[j]) return fail(BSGD_EINVAL, "col ranges must be nonempty and ascending");
    if (row_bounds[0] != 0 || col_bounds[0] != 0) return fail(BSGD_EINVAL, "ranges must start at 0");
    if (row_bounds[num_row_blocks] != rows || col_bounds[num_col_blocks] != cols)
        return fail(BSGD_EINVAL, "partition covers %lldx%lld, matrix is %lldx%lld",
                    (long long)row_bounds[num_row_blocks], (long long)col_bounds[num_col_blocks],
                    (long long)rows, (long long)cols);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(BSGD_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(BSGD_EINVAL, "device %d out of range", device);
    return BSGD_OK;
}

static bsgd_plan *plan_new(int device, int64_t rows, int64_t cols, int64_t nnz, int value_dtype, int64_t M,
                           int64_t N, const int64_t *row_bounds, const int64_t *col_bounds) {
    bsgd_plan *p = new bsgd_plan();
    p->device = device;
    p->rows = rows; p->cols = cols; p->nnz = nnz; p->vdt = value_dtype;
    p->M = M; p->N = N;
    p->row_bounds.assign(row_bounds, row_bounds + M + 1);
    p->col_bounds.assign(col_bounds, col_bounds + N + 1);
    p->srows = rows; p->scols = cols; p->snnz = nnz;
    const double mean_r = (double)nnz / rows, mean_c = (double)nnz / cols;
    // lanes per row: short rows take 8-16 entries per lane through 16-byte loads
    // (configs[1]: 32-nnz rows G = 4, 0.291 -> 0.267 ms; 128-nnz columns G = 8,
    // 0.289 -> 0.277 ms, tools/gsweep.py), long rows (CT) a full warp
    auto pick = [](double mean) { return mean < 48.0 ? 4 : (mean < 256.0 ? 8 : 32); };
    p->g_fwd = pick(mean_r);
    p->g_tr = pick(mean_c);
    auto lanes = [](const char *e) { const int v = atoi(e); return (v == 4 || v == 8) ? v : 32; };
    if (const char *e = getenv("BSGD_G_TR")) p->g_tr = lanes(e);   // experiments
    if (const char *e = getenv("BSGD_G_FWD")) p->g_fwd = lanes(e);
    return p;
}

// depth > 1: slice-stacked plan, (rows, cols, nnz) describe the stored A2
static int stacked_check(int64_t depth, int64_t rows, int64_t cols) {
    if (depth < 2) return fail(BSGD_EINVAL, "depth must be >= 2 (a single slice is an ordinary plan)");
    if (rows > (((int64_t)1 << 31) - 1) / depth || cols > (((int64_t)1 << 31) - 1) / depth)
        return fail(BSGD_EINVAL, "stacked dimensions must be < 2^31");
    return BSGD_OK;
}

static void stacked_setup(bsgd_plan *p, int64_t depth, int64_t rows2, int64_t cols2, int64_t nnz2) {
    p->depth = depth;
    p->srows = rows2; p->scols = cols2; p->snnz = nnz2;
    int L = 1;
    while (L < 32 && L < depth) L <<= 1;
    p->lanes = L;
    // slices per chunk: keep (vector rows) x (chunk) x 8 bytes <= ~64 MB of L2
    int64_t budget = 64000000;
    if (const char *env = getenv("BSGD_STK_L2_BYTES")) budget = std::max<int64_t>(1, atoll(env));
    auto pick = [&](int64_t vec_rows) {
        const int64_t zc_max = std::max<int64_t>(1, budget / (vec_rows * 8));
        int kz = 4;
        while (kz > 1 && ((int64_t)L * kz > zc_max || (int64_t)L * (kz / 2) >= depth)) kz /= 2;
        // two slices per lane at least when the depth allows: one entry load and
        // block test then serve two products (configs[4] A^T: 6.8 -> 5.1 ms, the
        // larger working set still mostly hits L2; tools/stk_sweep.py)
        if (kz == 1 && (int64_t)L * 2 <= depth) kz = 2;
        return kz;
    };
    p->kz_fwd = pick(cols2);
    p->kz_tr = pick(rows2);
}

static int plan_create_host(bsgd_plan **out, int device, int64_t depth, int64_t rows, int64_t cols, int64_t nnz,
                            const int64_t *indptr, const int32_t *indices, const void *values, int value_dtype,
                            int64_t num_row_blocks, int64_t num_col_blocks, const int64_t *row_bounds,
                            const int64_t *col_bounds, void *stream) {
    if (!out) return fail(BSGD_EINVAL, "out is NULL");
    *out = nullptr;
    int rc = depth > 1 ? stacked_check(depth, rows, cols) : BSGD_OK;
    if (rc) return rc;
    rc = plan_args_check(rows * depth, cols * depth, nnz, value_dtype, num_row_blocks, num_col_blocks, row_bounds,
                         col_bounds, device);
    if (rc) return rc;
    if (!indptr || !indices || !values) return fail(BSGD_EINVAL, "NULL array");
    if (indptr[0] != 0 || indptr[rows] != nnz) return fail(BSGD_EINVAL, "indptr must run from 0 to nnz");
    DeviceGuard guard(device);
    cudaStream_t st = (cudaStream_t)stream;
    bsgd_plan *p = plan_new(device, rows * depth, cols * depth, nnz * depth, value_dtype, num_row_blocks,
                            num_col_blocks, row_bounds, col_bounds);
    if (depth > 1) stacked_setup(p, depth, rows, cols, nnz);
    else { p->srows = rows; p->scols = cols; p->snnz = nnz; }
    const size_t vb = (size_t)value_dtype;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&p->f_ptr, sizeof(int64_t) * (rows + 1));
    if (e == cudaSuccess) e = cudaMalloc(&p->f_idx, sizeof(int32_t) * nnz);
    if (e == cudaSuccess) e = cudaMalloc(&p->f_val, vb * nnz);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->f_ptr, indptr, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->f_idx, indices, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->f_val, values, vb * nnz, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
        plan_free(p);
        return fail(e == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA, "plan upload failed: %s",
                    cudaGetErrorString(e));
    }
    rc = plan_finish(p, st);
    if (rc) { plan_free(p); return rc; }
    *out = p;
    return BSGD_OK;
}

static int plan_create_adopt(bsgd_plan **out, int device, int64_t depth, int64_t rows, int64_t cols, int64_t nnz,
                             int64_t *indptr, int32_t *indices, void *values, int value_dtype,
                             int64_t num_row_blocks, int64_t num_col_blocks, const int64_t *row_bounds,
                             const int64_t *col_bounds, void *stream) {
    if (!out) return fail(BSGD_EINVAL, "out is NULL");
    *out = nullptr;
    int rc = depth > 1 ? stacked_check(depth, rows, cols) : BSGD_OK;
    if (rc) return rc;
    rc = plan_args_check(rows * depth, cols * depth, nnz, value_dtype, num_row_blocks, num_col_blocks, row_bounds,
                         col_bounds, device);
    if (rc) return rc;
    if (!indptr || !indices || !values) return fail(BSGD_EINVAL, "NULL array");
    DeviceGuard guard(device);
    cudaStream_t st = (cudaStream_t)stream;
    int64_t ends[2] = {-1, -1};
    CU(cudaMemcpyAsync(&ends[0], indptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(&ends[1], indptr + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (ends[0] != 0 || ends[1] != nnz) return fail(BSGD_EINVAL, "indptr must run from 0 to nnz");
    bsgd_plan *p = plan_new(device, rows * depth, cols * depth, nnz * depth, value_dtype, num_row_blocks,
                            num_col_blocks, row_bounds, col_bounds);
    if (depth > 1) stacked_setup(p, depth, rows, cols, nnz);
    else { p->srows = rows; p->scols = cols; p->snnz = nnz; }
    p->f_ptr = indptr;   // adopted: freed with the plan
    p->f_idx = indices;
    p->f_val = values;
    rc = plan_finish(p, st);
    if (rc) { plan_free(p); return rc; }
    *out = p;
    return BSGD_OK;
}

int bsgd_plan_create(bsgd_plan **out, int device, int64_t rows, int64_t cols, int64_t nnz,
                     const int64_t *indptr, const int32_t *indices, const void *values, int value_dtype,
                     int64_t num_row_blocks, int64_t num_col_blocks, const int64_t *row_bounds,
                     const int64_t *col_bounds, void *stream) {
    return plan_create_host(out, device, 1, rows, cols, nnz, indptr, indices, values, value_dtype, num_row_blocks,
                            num_col_blocks, row_bounds, col_bounds, stream);
}

int bsgd_plan_create_device(bsgd_plan **out, int device, int64_t rows, int64_t cols, int64_t nnz, int64_t *indptr,
                            int32_t *indices, void *values, int value_dtype, int64_t num_row_blocks,
                            int64_t num_col_blocks, const int64_t *row_bounds, const int64_t *col_bounds,
                            void *stream) {
    return plan_create_adopt(out, device, 1, rows, cols, nnz, indptr, indices, values, value_dtype, num_row_blocks,
                             num_col_blocks, row_bounds, col_bounds, stream);
}

int bsgd_plan_create_stacked(bsgd_plan **out, int device, int64_t depth, int64_t rows2, int64_t cols2, int64_t nnz2,
                             const int64_t *indptr, const int32_t *indices, const void *values, int value_dtype,
                             int64_t num_row_blocks, int64_t num_col_blocks, const int64_t *row_bounds,
                             const int64_t *col_bounds, void *stream) {
    if (depth < 2) return fail(BSGD_EINVAL, "depth must be >= 2 (a single slice is an ordinary plan)");
    return plan_create_host(out, device, depth, rows2, cols2, nnz2, indptr, indices, values, value_dtype,
                            num_row_blocks, num_col_blocks, row_bounds, col_bounds, stream);
}

int bsgd_plan_create_stacked_device(bsgd_plan **out, int device, int64_t depth, int64_t rows2, int64_t cols2,
                                    int64_t nnz2, int64_t *indptr, int32_t *indices, void *values, int value_dtype,
                                    int64_t num_row_blocks, int64_t num_col_blocks, const int64_t *row_bounds,
                                    const int64_t *col_bounds, void *stream) {
    if (depth < 2) return fail(BSGD_EINVAL, "depth must be >= 2 (a single slice is an ordinary plan)");
    return plan_create_adopt(out, device, depth, rows2, cols2, nnz2, indptr, indices, values, value_dtype,
                             num_row_blocks, num_col_blocks, row_bounds, col_bounds, stream);
}

int bsgd_plan_gather_tiles(bsgd_plan *p, int transposed, int64_t ntiles, const int64_t *tile_ptr,
                           const int64_t *tile_rows, void *stream) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (p->stacked()) return fail(BSGD_EINVAL, "stacked plans use bsgd_plan_stacked_tiles");
    DeviceGuard guard(p->device);
    bsgd_plan::GTileStore &S = transposed ? p->gt : p->gf;
    if (ntiles == 0) {
        p->device_bytes -= S.bytes;
        gtiles_free(S);
        return BSGD_OK;
    }
    if (ntiles < 0 || !tile_ptr || !tile_rows) return fail(BSGD_EINVAL, "bad tile arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int rc = p->vdt == BSGD_F32 ? build_gtiles<float>(p, transposed != 0, ntiles, tile_ptr, tile_rows, st)
                                : build_gtiles<double>(p, transposed != 0, ntiles, tile_ptr, tile_rows, st);
    if (rc) return rc;
    if (transposed) {   // the latest explicit request wins over a blocked copy of A^T
        p->device_bytes -= p->tb.bytes;
        blk_free(p->tb);
    }
    // The caller asked for these tiles, so they are kept: no timing race decides
    // which kernel a plan runs.  BlockOperator requests them where they win
    // (pixel rows of A^T for CT: 6.1 -> 4.2 ms at 1024^2, whose CSR gathers have
    // no sector locality) and not where they lose (ray rows of A: 4.5 -> 6.3 ms).
    (void)st;
    return BSGD_OK;
}

int bsgd_plan_blocked_transposed(bsgd_plan *p, int64_t grid_h, int64_t grid_w, void *stream) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (p->stacked()) return fail(BSGD_EINVAL, "stacked plans have no blocked stream");
    DeviceGuard guard(p->device);
    if (grid_h < 0 || grid_w < 0) {   // remove
        p->device_bytes -= p->tb.bytes;
        blk_free(p->tb);
        return BSGD_OK;
    }
    if ((grid_h || grid_w) && grid_h * grid_w != p->rows)
        return fail(BSGD_EINVAL, "grid %lld x %lld does not match the %lld rows of A", (long long)grid_h,
                    (long long)grid_w, (long long)p->rows);
    if (p->cols == 0 || p->nnz == 0) return BSGD_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = p->vdt == BSGD_F32 ? build_blocked_dir<float>(p, true, (int)grid_h, (int)grid_w, st)
                                : build_blocked_dir<double>(p, true, (int)grid_h, (int)grid_w, st);
    if (rc) return rc;
    return p->vdt == BSGD_F32 ? tune_blocked<float>(p, p->tb) : tune_blocked<double>(p, p->tb);
}

int bsgd_plan_stacked_tiles(bsgd_plan *p, int transposed, int64_t ntiles, const int64_t *tile_ptr,
                            const int64_t *tile_rows, void *stream) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (!p->stacked()) return fail(BSGD_EINVAL, "tiles apply to slice-stacked plans only");
    DeviceGuard guard(p->device);
    bsgd_plan::StkTileStore &S = transposed ? p->stt : p->sf;
    if (ntiles == 0) {
        p->device_bytes -= S.bytes;
        stk_tiles_free(S);
        return BSGD_OK;
    }
    if (ntiles < 0 || !tile_ptr || !tile_rows) return fail(BSGD_EINVAL, "bad tile arguments");
    cudaStream_t st = (cudaStream_t)stream;
    return p->vdt == BSGD_F32 ? build_stk_tiles<float>(p, transposed != 0, ntiles, tile_ptr, tile_rows, st)
                              : build_stk_tiles<double>(p, transposed != 0, ntiles, tile_ptr, tile_rows, st);
}

int bsgd_plan_stacked_info(const bsgd_plan *p, int64_t *depth, int64_t *rows2, int64_t *cols2, int64_t *nnz2) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (depth) *depth = p->depth;
    if (rows2) *rows2 = p->srows;
    if (cols2) *cols2 = p->scols;
    if (nnz2) *nnz2 = p->snnz;
    return BSGD_OK;
}

int bsgd_siddon_csr(int device, int64_t n, int64_t num_angles, int64_t num_bins, const double *cos_host,
                    const double *sin_host, int value_dtype, int64_t **indptr_out, int32_t **indices_out,
                    void **values_out, int64_t *nnz_out, void *stream) {
    if (n < 1 || num_angles < 1 || num_bins < 1 || !cos_host || !sin_host || !indptr_out || !indices_out ||
        !values_out || !nnz_out)
        return fail(BSGD_EINVAL, "bad siddon arguments");
    if (n * n >= ((int64_t)1 << 31)) return fail(BSGD_EINVAL, "image too large for int32 column indices");
    if (value_dtype != BSGD_F32 && value_dtype != BSGD_F64) return fail(BSGD_EINVAL, "value dtype must be 4 or 8");
    DeviceGuard guard(device);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nrays = num_angles * num_bins;
    double *ct = nullptr, *sn = nullptr;
    int64_t *counts = nullptr, *indptr = nullptr;
    int32_t *idx = nullptr;
    void *vals = nullptr, *temp = nullptr;
    size_t temp_bytes = 0;
    int rc = BSGD_OK;
    auto cleanup = [&]() { cudaFree(ct); cudaFree(sn); cudaFree(counts); cudaFree(temp); };
#define STRY(call)                                                                          \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) {                                                            \
            rc = fail(e_ == cudaErrorMemoryAllocation ? BSGD_ENOMEM : BSGD_ECUDA,           \
                      "siddon: %s failed: %s", #call, cudaGetErrorString(e_));              \
            cleanup(); cudaFree(indptr); cudaFree(idx); cudaFree(vals);                     \
            return rc;                                                                      \
        }                                                                                   \
    } while (0)
    STRY(cudaMalloc(&ct, sizeof(double) * num_angles));
    STRY(cudaMalloc(&sn, sizeof(double) * num_angles));
    STRY(cudaMemcpyAsync(ct, cos_host, sizeof(double) * num_angles, cudaMemcpyHostToDevice, st));
    STRY(cudaMemcpyAsync(sn, sin_host, sizeof(double) * num_angles, cudaMemcpyHostToDevice, st));
    STRY(cudaMalloc(&counts, sizeof(int64_t) * (nrays + 1)));
    STRY(cudaMalloc(&indptr, sizeof(int64_t) * (nrays + 1)));
    RayGeom G{n, num_bins, nrays, ct, sn};
    siddon_count_kernel<<<grid_1d(nrays, 128), 128, 0, st>>>(G, counts);
    STRY(cudaMemsetAsync(counts + nrays, 0, sizeof(int64_t), st));
    STRY(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts, indptr, nrays + 1, st));
    STRY(cudaMalloc(&temp, temp_bytes));
    STRY(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, indptr, nrays + 1, st));
    int64_t nnz = 0;
    STRY(cudaMemcpyAsync(&nnz, indptr + nrays, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    STRY(cudaStreamSynchronize(st));
    STRY(cudaMalloc(&idx, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    STRY(cudaMalloc(&vals, (size_t)value_dtype * std::max<int64_t>(nnz, 1)));
    if (value_dtype == BSGD_F32)
        siddon_fill_kernel<float><<<grid_1d(nrays, 128), 128, 0, st>>>(G, indptr, idx, (float *)vals);
    else
        siddon_fill_kernel<double><<<grid_1d(nrays, 128), 128, 0, st>>>(G, indptr, idx, (double *)vals);
    STRY(cudaGetLastError());
    STRY(cudaStreamSynchronize(st));
#undef STRY
    cleanup();
    *indptr_out = indptr;
    *indices_out = idx;
    *values_out = vals;
    *nnz_out = nnz;
    return BSGD_OK;
}

int bsgd_device_free(void *ptr) {
    if (ptr) CU(cudaFree(ptr));
    return BSGD_OK;
}

// host expansion of a stacked plan's logical CSR (A or A^T) restricted to
// outputs [o0, o1) and entries [e0, e1): test / inspection paths only
static int stacked_expand(const bsgd_plan *p, bool tr, int64_t o0, int64_t o1, int64_t e0, int64_t e1,
                          int64_t *indptr_out, int32_t *indices_out, void *values_out, cudaStream_t st) {
    const int64_t nr = tr ? p->scols : p->srows, D = p->depth, vb = p->vdt;
    std::vector<int64_t> ptr(nr + 1);
    std::vector<int32_t> idx(p->snnz);
    std::vector<char> val((size_t)p->snnz * vb);
    CU(cudaMemcpyAsync(ptr.data(), tr ? p->t_ptr : p->f_ptr, sizeof(int64_t) * (nr + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(idx.data(), tr ? p->t_idx : p->f_idx, sizeof(int32_t) * p->snnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(val.data(), tr ? p->t_val : p->f_val, (size_t)p->snnz * vb, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    int64_t w = 0;
    indptr_out[0] = 0;
    for (int64_t O = o0; O < o1; ++O) {
        const int64_t r = O / D, z = O - r * D;
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int64_t E = (int64_t)idx[k] * D + z;
            if (E >= e1) break;
            if (E < e0) continue;
            indices_out[w] = (int32_t)(E - e0);
            memcpy((char *)values_out + (size_t)w * vb, val.data() + (size_t)k * vb, vb);
            ++w;
        }
        indptr_out[O - o0 + 1] = w;
    }
    return BSGD_OK;
}

int bsgd_plan_csr_copy(const bsgd_plan *p, int64_t *indptr_out, int32_t *indices_out, void *values_out, void *stream) {
    if (!p || !indptr_out || !indices_out || !values_out) return fail(BSGD_EINVAL, "NULL argument");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->stacked()) return stacked_expand(p, false, 0, p->rows, 0, p->cols, indptr_out, indices_out, values_out, st);
    CU(cudaMemcpyAsync(indptr_out, p->f_ptr, sizeof(int64_t) * (p->rows + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(indices_out, p->f_idx, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(values_out, p->f_val, (size_t)p->vdt * p->nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return BSGD_OK;
}

int bsgd_plan_destroy(bsgd_plan *plan) {
    plan_free(plan);
    return BSGD_OK;
}

// The kernels launch_fwd / launch_tr dispatch to for this plan (same decision order).
static void kernel_choice(const bsgd_plan *p, bool tr, int32_t *kind, int32_t *lanes) {
    if (p->stacked()) {
        const bsgd_plan::StkTileStore &S = tr ? p->stt : p->sf;
        if (stk_tiles_used(p, S)) {
            *kind = BSGD_K_STACKED_TILE;
            *lanes = S.kz;
        } else {
            *kind = BSGD_K_STACKED;
            *lanes = tr ? p->kz_tr : p->kz_fwd;
        }
        return;
    }
    if (tr && blocked_tr_on(p)) {
        *kind = p->tb.half ? BSGD_K_BLOCKED_CMP : BSGD_K_BLOCKED;
        *lanes = p->tb.gb;
        return;
    }
    const bsgd_plan::GTileStore &G = tr ? p->gt : p->gf;
    if (gtiles_on(G)) {
        *kind = BSGD_K_GTILE;
        *lanes = 16;
        return;
    }
    if (!tr && blocked_on(p)) {
        *kind = p->fb.half ? BSGD_K_BLOCKED_CMP : BSGD_K_BLOCKED;
        *lanes = p->fb.gb;
        return;
    }
    *kind = BSGD_K_CSR;
    *lanes = tr ? p->g_tr : p->g_fwd;
}

int bsgd_plan_kernel_info(const bsgd_plan *p, bsgd_kernel_info *out) {
    if (!p || !out) return fail(BSGD_EINVAL, "NULL argument");
    *out = bsgd_kernel_info{};
    kernel_choice(p, false, &out->fwd_kernel, &out->fwd_lanes);
    kernel_choice(p, true, &out->tr_kernel, &out->tr_lanes);
    out->depth = p->depth;
    out->fwd_order = (!p->stacked() && blocked_on(p) && !gtiles_on(p->gf)) ? p->fb.order : 0;
    out->tr_order = (!p->stacked() && blocked_tr_on(p)) ? p->tb.order : 0;
    return BSGD_OK;
}

int bsgd_plan_set_timing(bsgd_plan *p, int enable) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    p->timing.on = enable != 0;
    p->timing.used = 0;
    return BSGD_OK;
}

int bsgd_plan_timing(bsgd_plan *p, double *ms_out, int64_t *epochs_out) {
    if (!p || !ms_out) return fail(BSGD_EINVAL, "NULL argument");
    DeviceGuard guard(p->device);
    bsgd_plan::Timing &T = p->timing;
    for (int k = 0; k < BSGD_TIMING_PHASES; ++k) ms_out[k] = 0.0;
    const size_t epochs = T.used / kPhaseEvents;
    if (epochs) {
        cudaError_t e = cudaEventSynchronize(T.pool[T.used - 1]);
        for (size_t q = 0; q < epochs && e == cudaSuccess; ++q) {
            const cudaEvent_t *ev = &T.pool[q * kPhaseEvents];
            for (int k = 0; k < BSGD_TIMING_PHASES && e == cudaSuccess; ++k) {
                float ms = 0.f;
                e = cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
                ms_out[k] += ms;
            }
        }
        if (e != cudaSuccess) return fail(BSGD_ECUDA, "phase timing: %s", cudaGetErrorString(e));
    }
    if (epochs_out) *epochs_out = (int64_t)epochs;
    T.used = 0;
    return BSGD_OK;
}

int bsgd_plan_info(const bsgd_plan *p, int64_t *rows, int64_t *cols, int64_t *nnz, int *value_dtype,
                   int64_t *device_bytes) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (rows) *rows = p->rows;
    if (cols) *cols = p->cols;
    if (nnz) *nnz = p->nnz;
    if (value_dtype) *value_dtype = p->vdt;
    if (device_bytes) *device_bytes = (int64_t)p->device_bytes;
    return BSGD_OK;
}

static int check_block(const bsgd_plan *p, int64_t i, int64_t j) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (i < 0 || i >= p->M || j < 0 || j >= p->N)
        return fail(BSGD_EINVAL, "block (%lld, %lld) outside the %lldx%lld grid", (long long)i, (long long)j,
                    (long long)p->M, (long long)p->N);
    return BSGD_OK;
}

int bsgd_plan_block_nnz(const bsgd_plan *p, int64_t i, int64_t j, int64_t *out) {
    int rc = check_block(p, i, j);
    if (rc) return rc;
    if (!out) return fail(BSGD_EINVAL, "out is NULL");
    *out = p->block_nnz[i * p->N + j];
    return BSGD_OK;
}

int bsgd_plan_block_copy(const bsgd_plan *p, int64_t i, int64_t j, int64_t *indptr_out, int32_t *indices_out,
                         void *values_out, void *stream) {
    int rc = check_block(p, i, j);
    if (rc) return rc;
    if (!indptr_out || !indices_out || !values_out) return fail(BSGD_EINVAL, "NULL output");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t r0 = p->row_bounds[i], r1 = p->row_bounds[i + 1];
    const int64_t c0 = p->col_bounds[j], c1 = p->col_bounds[j + 1];
    if (p->stacked()) return stacked_expand(p, false, r0, r1, c0, c1, indptr_out, indices_out, values_out, st);
    std::vector<int64_t> ptr(r1 - r0 + 1);
    CU(cudaMemcpyAsync(ptr.data(), p->f_ptr + r0, sizeof(int64_t) * (r1 - r0 + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const int64_t base = ptr[0], len = ptr[r1 - r0] - base;
    std::vector<int32_t> idx(len);
    std::vector<char> val((size_t)len * p->vdt);
    if (len > 0) {
        CU(cudaMemcpyAsync(idx.data(), p->f_idx + base, sizeof(int32_t) * len, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(val.data(), (const char *)p->f_val + (size_t)base * p->vdt, (size_t)len * p->vdt,
                           cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    int64_t w = 0;
    indptr_out[0] = 0;
    for (int64_t r = 0; r < r1 - r0; ++r) {
        const int32_t *b = idx.data() + (ptr[r] - base), *e = idx.data() + (ptr[r + 1] - base);
        const int32_t *lo = std::lower_bound(b, e, (int32_t)c0);
        const int32_t *hi = std::lower_bound(lo, e, (int32_t)c1);
        for (const int32_t *q = lo; q < hi; ++q, ++w) {
            indices_out[w] = *q - (int32_t)c0;
            memcpy((char *)values_out + (size_t)w * p->vdt, val.data() + (size_t)(q - idx.data()) * p->vdt, p->vdt);
        }
        indptr_out[r + 1] = w;
    }
    return BSGD_OK;
}

int bsgd_plan_transpose_copy(const bsgd_plan *p, int64_t *indptr_out, int32_t *indices_out, void *values_out,
                             void *stream) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    if (!indptr_out || !indices_out || !values_out) return fail(BSGD_EINVAL, "NULL output");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->stacked()) return stacked_expand(p, true, 0, p->cols, 0, p->rows, indptr_out, indices_out, values_out, st);
    CU(cudaMemcpyAsync(indptr_out, p->t_ptr, sizeof(int64_t) * (p->cols + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(indices_out, p->t_idx, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(values_out, p->t_val, (size_t)p->vdt * p->nnz, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return BSGD_OK;
}

int bsgd_block_matvec(const bsgd_plan *p, int64_t i, int64_t j, const double *x_j, double *out, void *stream) {
    int rc = check_block(p, i, j);
    if (rc) return rc;
    if (!x_j || !out) return fail(BSGD_EINVAL, "NULL vector");
    DeviceGuard guard(p->device);
    const int64_t r0 = p->row_bounds[i], r1 = p->row_bounds[i + 1];
    const int64_t c0 = p->col_bounds[j], c1 = p->col_bounds[j + 1];
    if (p->stacked()) {
        const int g = grid_1d(r1 - r0);
        if (p->vdt == BSGD_F32)
            stacked_block_kernel<float><<<g, kThreads, 0, (cudaStream_t)stream>>>(
                p->f_ptr, p->f_idx, (const float *)p->f_val, p->depth, r0, r1, c0, c1, x_j, out);
        else
            stacked_block_kernel<double><<<g, kThreads, 0, (cudaStream_t)stream>>>(
                p->f_ptr, p->f_idx, (const double *)p->f_val, p->depth, r0, r1, c0, c1, x_j, out);
        LAUNCHED();
        return BSGD_OK;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(r1 - r0, kThreads / 32), num_sms() * 8));
    if (p->vdt == BSGD_F32)
        block_seg_kernel<float><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p->f_ptr, p->f_idx, (const float *)p->f_val,
                                                                            r0, r1, c0, c1, x_j, out);
    else
        block_seg_kernel<double><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p->f_ptr, p->f_idx, (const double *)p->f_val,
                                                                             r0, r1, c0, c1, x_j, out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_block_matvec_transpose(const bsgd_plan *p, int64_t i, int64_t j, const double *r_i, double *out,
                                void *stream) {
    int rc = check_block(p, i, j);
    if (rc) return rc;
    if (!r_i || !out) return fail(BSGD_EINVAL, "NULL vector");
    DeviceGuard guard(p->device);
    const int64_t r0 = p->row_bounds[i], r1 = p->row_bounds[i + 1];
    const int64_t c0 = p->col_bounds[j], c1 = p->col_bounds[j + 1];
    if (p->stacked()) {
        const int g = grid_1d(c1 - c0);
        if (p->vdt == BSGD_F32)
            stacked_block_kernel<float><<<g, kThreads, 0, (cudaStream_t)stream>>>(
                p->t_ptr, p->t_idx, (const float *)p->t_val, p->depth, c0, c1, r0, r1, r_i, out);
        else
            stacked_block_kernel<double><<<g, kThreads, 0, (cudaStream_t)stream>>>(
                p->t_ptr, p->t_idx, (const double *)p->t_val, p->depth, c0, c1, r0, r1, r_i, out);
        LAUNCHED();
        return BSGD_OK;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(c1 - c0, kThreads / 32), num_sms() * 8));
    // A^T rows [c0, c1), entries with A-row index in [r0, r1)
    if (p->vdt == BSGD_F32)
        block_seg_kernel<float><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p->t_ptr, p->t_idx, (const float *)p->t_val,
                                                                            c0, c1, r0, r1, r_i, out);
    else
        block_seg_kernel<double><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p->t_ptr, p->t_idx, (const double *)p->t_val,
                                                                             c0, c1, r0, r1, r_i, out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_matvec(const bsgd_plan *p, const double *x, double *out, void *stream) {
    if (!p || !x || !out) return fail(BSGD_EINVAL, "NULL argument");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    return DISPATCH_V(p, launch_fwd<V>(p, x, EpiStore{out, 1.0}, nullptr, nullptr, st));
}

int bsgd_rmatvec(const bsgd_plan *p, const double *w, double *out, void *stream) {
    if (!p || !w || !out) return fail(BSGD_EINVAL, "NULL argument");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    return DISPATCH_V(p, launch_tr<V>(p, w, EpiStore{out, 1.0}, nullptr, nullptr, st));
}

int bsgd_grad(const bsgd_plan *p, const double *r, double *g, void *stream) {
    if (!p || !r || !g) return fail(BSGD_EINVAL, "NULL argument");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    return DISPATCH_V(p, launch_tr<V>(p, r, EpiStore{g, 2.0}, nullptr, nullptr, st));
}

int bsgd_residual(const bsgd_plan *p, const double *x, const double *y, double *r_out, double *sumsq_out,
                  void *scratch, void *stream) {
    if (!p || !x || !y || !r_out) return fail(BSGD_EINVAL, "NULL argument");
    if (sumsq_out && !scratch) return fail(BSGD_EINVAL, "scratch required for sumsq_out");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    double *part = sumsq_out ? (double *)scratch : nullptr;
    int64_t *cnt = sumsq_out ? (int64_t *)((char *)scratch + sizeof(double) * kMaxPartials) : nullptr;
    EpiResid e{y, r_out};
    int rc = DISPATCH_V(p, launch_fwd<V>(p, x, e, part, cnt, st));
    if (rc) return rc;
    if (sumsq_out) {
        sum_counted_kernel<<<1, 32, 0, st>>>(part, cnt, sumsq_out);
        LAUNCHED();
    }
    return BSGD_OK;
}

int bsgd_assemble_residual(int64_t rows, int64_t num_col_blocks, const double *y, const double *z_cache,
                           double *out, void *stream) {
    if (rows < 1 || num_col_blocks < 0 || !y || !out || (num_col_blocks > 0 && !z_cache))
        return fail(BSGD_EINVAL, "bad assemble_residual arguments");
    assemble_kernel<<<grid_1d(rows), kThreads, 0, (cudaStream_t)stream>>>(rows, num_col_blocks, y, z_cache, out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_pair_products(const bsgd_plan *p, int64_t n_rows_sel, const int64_t *row_sel, int64_t n_cols_sel,
                       const int64_t *col_sel, const double *x_k, const double *r_k, const double *y,
                       double *z_cache, double *g, double *r_next, void *stream) {
    if (!p || !x_k || !r_k || !y || !z_cache || !g || !r_next) return fail(BSGD_EINVAL, "NULL argument");
    if (p->M > 256 || p->N > 256) return fail(BSGD_EINVAL, "pair path supports at most 256 blocks per side");
    // a row-slab shard may own none of the selected row blocks (n_rows_sel = 0): its g is
    // zero and its residual is rebuilt from the unchanged cache
    if (n_rows_sel < 0 || n_cols_sel < 1 || (n_rows_sel > 0 && !row_sel) || !col_sel)
        return fail(BSGD_EINVAL, "alpha/gamma select no blocks");
    BlockMask rs{{0, 0, 0, 0}}, cs{{0, 0, 0, 0}};
    for (int64_t k = 0; k < n_rows_sel; ++k) {
        if (row_sel[k] < 0 || row_sel[k] >= p->M) return fail(BSGD_EINVAL, "row block index out of range");
        rs.w[row_sel[k] >> 6] |= 1ull << (row_sel[k] & 63);
    }
    for (int64_t k = 0; k < n_cols_sel; ++k) {
        if (col_sel[k] < 0 || col_sel[k] >= p->N) return fail(BSGD_EINVAL, "col block index out of range");
        cs.w[col_sel[k] >> 6] |= 1ull << (col_sel[k] & 63);
    }
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->stacked()) {
        const int gr = grid_1d(p->rows), gc = grid_1d(p->cols);
        if (p->vdt == BSGD_F32) {
            stacked_pair_grad_kernel<float><<<gc, kThreads, 0, st>>>(p->t_ptr, p->t_idx, (const float *)p->t_val,
                                                                     p->depth, p->cols, p->d_row_bounds, p->M,
                                                                     p->d_col_bounds, p->N, rs, cs, r_k, g);
            stacked_pair_forward_kernel<float><<<gr, kThreads, 0, st>>>(
                p->f_ptr, p->f_idx, (const float *)p->f_val, p->depth, p->rows, p->d_row_bounds, p->M,
                p->d_col_bounds, p->N, rs, cs, x_k, y, z_cache, r_next);
        } else {
            stacked_pair_grad_kernel<double><<<gc, kThreads, 0, st>>>(p->t_ptr, p->t_idx, (const double *)p->t_val,
                                                                      p->depth, p->cols, p->d_row_bounds, p->M,
                                                                      p->d_col_bounds, p->N, rs, cs, r_k, g);
            stacked_pair_forward_kernel<double><<<gr, kThreads, 0, st>>>(
                p->f_ptr, p->f_idx, (const double *)p->f_val, p->depth, p->rows, p->d_row_bounds, p->M,
                p->d_col_bounds, p->N, rs, cs, x_k, y, z_cache, r_next);
        }
        LAUNCHED();
        return BSGD_OK;
    }
    const int gr = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(p->rows, kThreads / 32), num_sms() * 8));
    const int gc = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(p->cols, kThreads / 32), num_sms() * 8));
    if (p->vdt == BSGD_F32) {
        pair_grad_kernel<float><<<gc, kThreads, 0, st>>>(p->t_ptr, p->t_idx, (const float *)p->t_val, p->cols,
                                                         p->d_row_bounds, p->M, p->d_col_bounds, p->N, rs, cs, r_k, g);
        pair_forward_kernel<float><<<gr, kThreads, 0, st>>>(p->f_ptr, p->f_idx, (const float *)p->f_val, p->rows,
                                                            p->d_row_bounds, p->M, p->d_col_bounds, p->N, rs, cs,
                                                            x_k, y, z_cache, r_next);
    } else {
        pair_grad_kernel<double><<<gc, kThreads, 0, st>>>(p->t_ptr, p->t_idx, (const double *)p->t_val, p->cols,
                                                          p->d_row_bounds, p->M, p->d_col_bounds, p->N, rs, cs, r_k, g);
        pair_forward_kernel<double><<<gr, kThreads, 0, st>>>(p->f_ptr, p->f_idx, (const double *)p->f_val, p->rows,
                                                             p->d_row_bounds, p->M, p->d_col_bounds, p->N, rs, cs,
                                                             x_k, y, z_cache, r_next);
    }
    LAUNCHED();
    return BSGD_OK;
}

// ---- TV ----
size_t bsgd_tv_prox_workspace_bytes(int64_t height, int64_t width) {
    if (height < 1 || width < 1) return 0;
    return ws_layout(nullptr, 1, height * width, nullptr);
}

size_t bsgd_tv_prox3_workspace_bytes(int64_t depth, int64_t height, int64_t width) {
    if (depth < 1 || height < 1 || width < 1) return 0;
    return ws_layout(nullptr, 1, depth * height * width, nullptr);
}

static int tv_prox_any(int64_t depth, int64_t height, int64_t width, const double *img, double *out, double weight,
                       int32_t max_inner_iters, double tol, void *workspace, size_t workspace_bytes,
                       bsgd_prox_info *info_out, double *dual_objectives, void *stream) {
    if (depth < 1 || height < 1 || width < 1) return fail(BSGD_EINVAL, "image dimensions must be positive");
    if (!img || !out) return fail(BSGD_EINVAL, "NULL image");
    if (!(weight >= 0.0)) return fail(BSGD_EINVAL, "prox weight must be nonnegative");
    if (max_inner_iters < 1) return fail(BSGD_EINVAL, "max_inner_iters must be >= 1");
    if (!(tol > 0.0)) return fail(BSGD_EINVAL, "tol must be positive");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = depth * height * width;
    if (weight == 0.0) {  // tv.py:190-193: identity, converged
        CU(cudaMemcpyAsync(out, img, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        if (info_out) {
            const bsgd_prox_info zero = {0, 1, 0, 0};
            static_assert(sizeof(bsgd_prox_info) == 16, "layout");
            set_info_kernel<<<1, 1, 0, st>>>((int32_t *)info_out, zero.iterations, zero.converged, zero.restarts,
                                             zero.fell_back);
            LAUNCHED();
        }
        return BSGD_OK;
    }
    Ws ws;
    const size_t need = ws_layout(workspace, 1, n, &ws);
    if (!workspace || workspace_bytes < need) return fail(BSGD_EINVAL, "workspace too small (%zu < %zu)", workspace_bytes, need);
    ProxArgs a = {};
    a.D = depth; a.H = height; a.W = width; a.N = n;
    a.b = img;
    prox_fields(a, ws, n);
    a.w = weight;
    a.step = 1.0 / ((depth > 1 ? 12.0 : 8.0) * weight);  // 1/(||D||^2 w): 8 in 2D (tv.py:195), 12 in 3D
    a.tol = tol;
    a.max_iters = max_inner_iters;
    a.out_img = out;
    a.scal = ws.scal;
    a.info = (int32_t *)info_out;
    a.dual = dual_objectives;
    return launch_prox(a, st);
}

int bsgd_tv_prox(int64_t height, int64_t width, const double *img, double *out, double weight,
                 int32_t max_inner_iters, double tol, void *workspace, size_t workspace_bytes,
                 bsgd_prox_info *info_out, double *dual_objectives, void *stream) {
    return tv_prox_any(1, height, width, img, out, weight, max_inner_iters, tol, workspace, workspace_bytes, info_out,
                       dual_objectives, stream);
}

int bsgd_tv_prox3(int64_t depth, int64_t height, int64_t width, const double *vol, double *out, double weight,
                  int32_t max_inner_iters, double tol, void *workspace, size_t workspace_bytes,
                  bsgd_prox_info *info_out, double *dual_objectives, void *stream) {
    if (depth < 2) return fail(BSGD_EINVAL, "bsgd_tv_prox3 needs depth >= 2 (use bsgd_tv_prox for images)");
    return tv_prox_any(depth, height, width, vol, out, weight, max_inner_iters, tol, workspace, workspace_bytes,
                       info_out, dual_objectives, stream);
}

static int reduce_launch(int64_t n, const double *a, const double *b, int mode, double *out, void *scratch,
                         cudaStream_t st) {
    if (n < 0 || !out || !scratch || (n > 0 && (!a || !b))) return fail(BSGD_EINVAL, "bad reduction arguments");
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, kThreads), std::min(num_sms() * 8, kMaxPartials)));
    double *part = (double *)scratch;
    dot_part_kernel<<<grid, kThreads, 0, st>>>(n, a, b, mode, part);
    sum_parts_kernel<<<1, 32, 0, st>>>(part, grid, out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_dot(int64_t n, const double *a, const double *b, double *out, void *scratch, void *stream) {
    return reduce_launch(n, a, b, 0, out, scratch, (cudaStream_t)stream);
}

int bsgd_sqdist(int64_t n, const double *a, const double *b, double *out, void *scratch, void *stream) {
    return reduce_launch(n, a, b, 1, out, scratch, (cudaStream_t)stream);
}

static int tv_value_any(int64_t depth, int64_t height, int64_t width, const double *img, double *out, void *scratch,
                        void *stream) {
    if (depth < 1 || height < 1 || width < 1 || !img || !out || !scratch) return fail(BSGD_EINVAL, "bad tv_value arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = depth * height * width;
    int ds = 0;
    int rc = pw_depth(n, &ds);
    if (rc) return rc;
    const int64_t S = (int64_t)1 << ds;
    const int G = (int)std::min<int64_t>(S, 256);
    if (S / G > kPwMaxQ * (kThreads / 8)) return fail(BSGD_EINVAL, "image too large for tv_value (%lld pixels)", (long long)n);
    if (depth > 1) tv_value_part_kernel<3><<<G, kThreads, 0, st>>>(depth, height, width, img, ds, (double *)scratch);
    else tv_value_part_kernel<2><<<G, kThreads, 0, st>>>(1, height, width, img, ds, (double *)scratch);
    pw_top_kernel<<<1, kThreads, 0, st>>>(ds, G, (const double *)scratch, out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_tv_value(int64_t height, int64_t width, const double *img, double *out, void *scratch, void *stream) {
    return tv_value_any(1, height, width, img, out, scratch, stream);
}

int bsgd_tv_value3(int64_t depth, int64_t height, int64_t width, const double *vol, double *out, void *scratch,
                   void *stream) {
    return tv_value_any(depth, height, width, vol, out, scratch, stream);
}

int bsgd_discrete_gradient(int64_t height, int64_t width, const double *img, double *dv, double *dh, void *stream) {
    if (height < 1 || width < 1 || !img || !dv || !dh) return fail(BSGD_EINVAL, "bad gradient arguments");
    gradient_kernel<<<grid_1d(height * width), kThreads, 0, (cudaStream_t)stream>>>(height, width, img, dv, dh);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_discrete_divergence(int64_t height, int64_t width, const double *pv, const double *ph, double *out,
                             void *stream) {
    if (height < 1 || width < 1 || !pv || !ph || !out) return fail(BSGD_EINVAL, "bad divergence arguments");
    divergence_kernel<<<grid_1d(height * width), kThreads, 0, (cudaStream_t)stream>>>(height, width, pv, ph, out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_discrete_gradient3(int64_t depth, int64_t height, int64_t width, const double *vol, double *dz, double *dv,
                            double *dh, void *stream) {
    if (depth < 1 || height < 1 || width < 1 || !vol || !dz || !dv || !dh)
        return fail(BSGD_EINVAL, "bad gradient arguments");
    gradient3_kernel<<<grid_1d(depth * height * width), kThreads, 0, (cudaStream_t)stream>>>(depth, height, width,
                                                                                           vol, dz, dv, dh);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_discrete_divergence3(int64_t depth, int64_t height, int64_t width, const double *pz, const double *pv,
                              const double *ph, double *out, void *stream) {
    if (depth < 1 || height < 1 || width < 1 || !pz || !pv || !ph || !out)
        return fail(BSGD_EINVAL, "bad divergence arguments");
    divergence3_kernel<<<grid_1d(depth * height * width), kThreads, 0, (cudaStream_t)stream>>>(depth, height, width,
                                                                                             pz, pv, ph, out);
    LAUNCHED();
    return BSGD_OK;
}

// ---- epoch ----
size_t bsgd_epoch_workspace_bytes(const bsgd_plan *p, int64_t height, int64_t width) {
    if (!p) return 0;
    // the prox fields are sized by the plan's columns (height*width, or
    // depth*height*width for volumes, must equal cols when lam > 0)
    const int64_t n = (height > 0 && width > 0) ? p->cols : 0;
    return ws_layout(nullptr, p->cols, n, nullptr);
}

static int check_epoch_args(int64_t cols, const bsgd_epoch_args *a, Ws *ws) {
    if (!a) return fail(BSGD_EINVAL, "args is NULL");
    if (!(a->mu > 0.0)) return fail(BSGD_EINVAL, "mu must be positive");
    if (a->lam < 0.0) return fail(BSGD_EINVAL, "lam must be nonnegative");
    const bool prox = a->lam > 0.0;
    if (prox) {
        const int64_t depth = a->depth > 1 ? a->depth : 1;
        if (a->height < 1 || a->width < 1 || depth * a->height * a->width != cols)
            return fail(BSGD_EINVAL, "layout required when lam > 0 (depth*height*width must equal cols)");
        if (a->max_inner_iters < 1) return fail(BSGD_EINVAL, "max_inner_iters must be >= 1");
        if (!(a->tol > 0.0)) return fail(BSGD_EINVAL, "tol must be positive");
    }
    if (!a->x_k || !a->g || !a->x_next) return fail(BSGD_EINVAL, "x_k, g and x_next are required");
    if (!a->workspace) return fail(BSGD_EINVAL, "workspace is NULL");
    const size_t need = ws_layout(a->workspace, cols, prox ? cols : 0, ws);
    if (a->workspace_bytes < need) return fail(BSGD_EINVAL, "workspace too small (%zu < %zu)", a->workspace_bytes, need);
    if (!(a->flags & BSGD_EP_NO_TAIL) && (!a->history || !a->epoch_counter))
        return fail(BSGD_EINVAL, "history and epoch_counter are required");
    if ((a->flags & BSGD_EP_MONITOR) && !a->f_curr) return fail(BSGD_EINVAL, "f_curr required with MONITOR");
    return BSGD_OK;
}

// x_next = prox(x_k + mu g) from a g already in memory (solvers.py:305-314)
static int run_step(int64_t cols, const bsgd_epoch_args *a, const Ws &ws, cudaStream_t st) {
    const bool prox = a->lam > 0.0;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(cols, kThreads), std::min(num_sms() * 8, kMaxPartials)));
    step_kernel<<<grid, kThreads, 0, st>>>(cols, a->x_k, a->g, a->mu, a->x_next, prox ? ws.uimg : nullptr, a->perm,
                                          a->x_true, ws.xpart, ws.ctl);
    LAUNCHED();
    return BSGD_OK;
}

static int run_prox(const bsgd_epoch_args *a, const Ws &ws, cudaStream_t st) {
    const int64_t depth = a->depth > 1 ? a->depth : 1;
    const int64_t n = depth * a->height * a->width;
    ProxArgs pa = {};
    pa.D = depth; pa.H = a->height; pa.W = a->width; pa.N = n;
    pa.b = ws.uimg;
    prox_fields(pa, ws, n);
    pa.w = a->mu * a->lam;  // tv.py weight = mu_try * cfg.lam (solvers.py:310)
    pa.step = 1.0 / ((depth > 1 ? 12.0 : 8.0) * pa.w);
    pa.tol = a->tol;
    pa.max_iters = a->max_inner_iters;
    pa.out_img = nullptr;
    pa.x_next = a->x_next; pa.perm = a->perm; pa.x_k = a->x_k; pa.g = a->g; pa.x_true = a->x_true;
    pa.xpart = ws.xpart; pa.nx = ws.ctl; pa.scal = ws.scal;
    pa.info = nullptr;
    pa.dual = a->dual_objectives;
    return launch_prox(pa, st);
}

static int run_tail(const bsgd_epoch_args *a, const Ws &ws, int fnext_mode, const double *fnext_dev, cudaStream_t st) {
    TailArgs t = {};
    t.ctl = ws.ctl; t.xpart = ws.xpart; t.rpart = ws.rpart; t.scal = ws.scal;
    t.fnext_dev = fnext_dev;
    t.fnext_mode = fnext_mode;
    t.monitor = (a->flags & BSGD_EP_MONITOR) ? 1 : 0;
    t.has_prox = a->lam > 0.0 ? 1 : 0;
    t.mu = a->mu;
    t.f_curr = a->f_curr;
    t.history = a->history;
    t.counter = a->epoch_counter;
    t.cap = a->history_capacity;
    tail_kernel<<<1, 32, 0, st>>>(t);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_epoch(const bsgd_plan *p, const bsgd_epoch_args *a, void *stream) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    Ws ws;
    int rc = check_epoch_args(p->cols, a, &ws);
    if (rc) return rc;
    const uint32_t fl = a->flags;
    if (!(fl & BSGD_EP_SKIP_GRAD) && !a->r_k) return fail(BSGD_EINVAL, "r_k is required");
    if ((fl & (BSGD_EP_R_NEXT | BSGD_EP_LOOKAHEAD)) && !a->y) return fail(BSGD_EINVAL, "y is required");
    if ((fl & BSGD_EP_R_NEXT) && !a->r_next) return fail(BSGD_EINVAL, "r_next is required");
    if ((fl & BSGD_EP_LOOKAHEAD) && !a->r_ahead) return fail(BSGD_EINVAL, "r_ahead is required");
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    EpochTimer timer(p, st);
#define TIMING_MARK(k) timer.mark(k)
    const bool prox = a->lam > 0.0;
    EpiStep es{a->g, a->x_k, a->mu, a->x_next, prox ? ws.uimg : nullptr, a->perm, a->x_true};
    if (fl & BSGD_EP_SKIP_GRAD) {
        rc = run_step(p->cols, a, ws, st);
        if (!rc && (fl & BSGD_EP_R_NEXT))
            rc = DISPATCH_V(p, launch_fwd<V>(p, a->x_k, EpiResid{a->y, a->r_next}, ws.rpart, ws.ctl + 2, st));
    } else {
        // K1(x_k) (when the lookahead r is invalid) then K2(r_k): both read the
        // snapshot x_k / r_k (solvers.py:281-290).  One merged grid was measured
        // slower on configs[1] (0.79 vs 0.66 ms per epoch; both halves are
        // gather-bound and the CTA split balances them poorly), so they run back to back.
        if (fl & BSGD_EP_R_NEXT)
            rc = DISPATCH_V(p, launch_fwd<V>(p, a->x_k, EpiResid{a->y, a->r_next}, ws.rpart, ws.ctl + 2, st));
        TIMING_MARK(1);
        if (!rc) {
            if (prox)   // the prox's output pass writes the step statistics
                rc = DISPATCH_V(p, launch_tr<V>(p, a->r_k, EpiStepImg{a->g, a->x_k, a->mu, ws.uimg, a->perm}, nullptr,
                                                nullptr, st));
            else
                rc = DISPATCH_V(p, launch_tr<V>(p, a->r_k, es, ws.xpart, ws.ctl, st));
        }
    }
    if (fl & BSGD_EP_SKIP_GRAD) TIMING_MARK(1);
    TIMING_MARK(2);
    if (rc) return rc;
    if (prox) {
        rc = run_prox(a, ws, st);
        if (rc) return rc;
    }
    TIMING_MARK(3);
    if (fl & BSGD_EP_LOOKAHEAD) {
        // K1(x_next): the next epoch's residual and the Eq. 9 monitor's f_next (solvers.py:319-320)
        rc = DISPATCH_V(p, launch_fwd<V>(p, a->x_next, EpiResid{a->y, a->r_ahead}, ws.rpart, ws.ctl + 1, st));
        if (rc) return rc;
    }
    TIMING_MARK(4);
    if (!(fl & BSGD_EP_NO_TAIL)) rc = run_tail(a, ws, (fl & BSGD_EP_LOOKAHEAD) ? 1 : 0, nullptr, st);
    TIMING_MARK(5);
#undef TIMING_MARK
    return rc;
}

int bsgd_step(int64_t cols, const bsgd_epoch_args *a, void *stream) {
    Ws ws;
    int rc = check_epoch_args(cols, a, &ws);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    rc = run_step(cols, a, ws, st);
    if (rc) return rc;
    if (a->lam > 0.0) rc = run_prox(a, ws, st);
    return rc;
}

int bsgd_epoch_forward(const bsgd_plan *p, const double *x, const double *y, double *r_out,
                       const bsgd_epoch_args *a, void *stream) {
    if (!p || !x || !y || !r_out || !a || !a->workspace) return fail(BSGD_EINVAL, "NULL argument");
    Ws ws;
    ws_layout(a->workspace, p->cols, a->lam > 0.0 ? p->cols : 0, &ws);
    DeviceGuard guard(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    return DISPATCH_V(p, launch_fwd<V>(p, x, EpiResid{y, r_out}, ws.rpart, ws.ctl + 1, st));
}

int bsgd_epoch_reduce_forward(const bsgd_plan *p, const bsgd_epoch_args *a, double *scalars_out, void *stream) {
    if (!p || !a || !a->workspace || !scalars_out) return fail(BSGD_EINVAL, "NULL argument");
    Ws ws;
    ws_layout(a->workspace, p->cols, a->lam > 0.0 ? p->cols : 0, &ws);
    sum_counted_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ws.rpart, ws.ctl + 1, scalars_out);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_epoch_tail(const bsgd_plan *p, const bsgd_epoch_args *a, const double *fnext_dev, void *stream) {
    if (!p) return fail(BSGD_EINVAL, "plan is NULL");
    Ws ws;
    int rc = check_epoch_args(p->cols, a, &ws);
    if (rc) return rc;
    if (!a->history || !a->epoch_counter) return fail(BSGD_EINVAL, "history and epoch_counter are required");
    return run_tail(a, ws, fnext_dev ? 2 : 0, fnext_dev, (cudaStream_t)stream);
}

// ---- slab-decomposed prox (multi-GPU) ----
size_t bsgd_slab_workspace_bytes(int64_t depth, int64_t height, int64_t width, int64_t count) {
    if (height < 1 || width < 1 || count < 1) return 0;
    int64_t off[BSGD_SLAB_SLOTS];
    return sizeof(double) * (size_t)slab_offsets(depth < 1 ? 1 : depth, height, width, count, off);
}

int bsgd_slab_layout(int64_t depth, int64_t height, int64_t width, int64_t count, int64_t *offsets_out,
                     int64_t *halo_out) {
    if (height < 1 || width < 1 || count < 1 || !offsets_out || !halo_out) return fail(BSGD_EINVAL, "bad slab layout query");
    slab_offsets(depth < 1 ? 1 : depth, height, width, count, offsets_out);
    *halo_out = slab_halo(depth < 1 ? 1 : depth, height, width);
    return BSGD_OK;
}

int bsgd_slab_step(const bsgd_slab *s, const double *x_k, const double *g, double mu, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c, false);
    if (rc) return rc;
    if (!x_k || !g) return fail(BSGD_EINVAL, "x_k and g are required");
    slab_step_kernel<<<c.grid, kThreads, 0, (cudaStream_t)stream>>>(c.v, x_k, g, mu);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_slab_init(const bsgd_slab *s, double *sums_out, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c);
    if (rc) return rc;
    if (!sums_out) return fail(BSGD_EINVAL, "sums_out is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    // p and q of both parities, halos included (tv.py:198-201)
    const int64_t len = s->count + 2 * slab_halo(c.v.a.D, s->height, s->width);
    int64_t off[BSGD_SLAB_SLOTS];
    slab_offsets(c.v.a.D, s->height, s->width, s->count, off);
    for (int slot = 1; slot <= 9; ++slot)
        if (off[slot] >= 0) CU(cudaMemsetAsync((double *)s->workspace + off[slot], 0, sizeof(double) * len, st));
    const size_t smem = 0;   // pw_cta_direct: no staging buffer
    if (c.dim == 3)
        return c.v.fast ? slab_sum_launch<2>(c, slab_init_kernel<3, true>, smem, sums_out, st)
                        : slab_sum_launch<2>(c, slab_init_kernel<3, false>, 0, sums_out, st);
    return c.v.fast ? slab_sum_launch<2>(c, slab_init_kernel<2, true>, smem, sums_out, st)
                    : slab_sum_launch<2>(c, slab_init_kernel<2, false>, 0, sums_out, st);
}

int bsgd_slab_candidate(const bsgd_slab *s, int32_t from_p, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (c.dim == 3) slab_candidate_kernel<3><<<c.grid, kThreads, 0, st>>>(c.v, from_p ? 1 : 0);
    else slab_candidate_kernel<2><<<c.grid, kThreads, 0, st>>>(c.v, from_p ? 1 : 0);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_slab_dual(const bsgd_slab *s, double beta, double *sums_out, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c);
    if (rc) return rc;
    if (!sums_out) return fail(BSGD_EINVAL, "sums_out is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    if (c.dim == 3) {
        const size_t smem = c.v.fast ? sizeof(double) * 7 * 8 * 128 : 0;
        auto kern = c.v.fast ? slab_dual_kernel<3, true> : slab_dual_kernel<3, false>;
        if (smem > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<c.G, kThreads, smem, st>>>(c.v, beta, c.part);
        slab_top_kernel<7><<<1, kThreads, 0, st>>>(c.v.ds, c.G, c.part, sums_out);
    } else {
        const size_t smem = c.v.fast ? sizeof(double) * 5 * 8 * 128 : 0;
        auto kern = c.v.fast ? slab_dual_kernel<2, true> : slab_dual_kernel<2, false>;
        if (smem > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<c.G, kThreads, smem, st>>>(c.v, beta, c.part);
        slab_top_kernel<5><<<1, kThreads, 0, st>>>(c.v.ds, c.G, c.part, sums_out);
    }
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_slab_finalize(const bsgd_slab *s, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (c.dim == 3) slab_finalize_kernel<3><<<c.grid, kThreads, 0, st>>>(c.v);
    else slab_finalize_kernel<2><<<c.grid, kThreads, 0, st>>>(c.v);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_slab_energy(const bsgd_slab *s, double *sums_out, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c);
    if (rc) return rc;
    if (!sums_out) return fail(BSGD_EINVAL, "sums_out is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t smem = 0;   // pw_cta_direct: no staging buffer
    if (c.dim == 3)
        return c.v.fast ? slab_sum_launch<2>(c, slab_energy_kernel<3, true>, smem, sums_out, st)
                        : slab_sum_launch<2>(c, slab_energy_kernel<3, false>, 0, sums_out, st);
    return c.v.fast ? slab_sum_launch<2>(c, slab_energy_kernel<2, true>, smem, sums_out, st)
                    : slab_sum_launch<2>(c, slab_energy_kernel<2, false>, 0, sums_out, st);
}

int bsgd_slab_output(const bsgd_slab *s, int32_t fell_back, double *x_next, const double *x_k, const double *g,
                     const double *x_true, double *stats_out, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c, false);
    if (rc) return rc;
    if (!x_next || !x_k || !g || !stats_out) return fail(BSGD_EINVAL, "x_next, x_k, g and stats_out are required");
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = std::min(c.grid, kSlabPartials / 4);
    if (c.dim == 3) slab_output_kernel<3><<<grid, kThreads, 0, st>>>(c.v, fell_back ? 1 : 0, x_next, x_k, g, x_true, c.part);
    else slab_output_kernel<2><<<grid, kThreads, 0, st>>>(c.v, fell_back ? 1 : 0, x_next, x_k, g, x_true, c.part);
    slab_sum4_kernel<<<1, 32, 0, st>>>(c.part, grid, stats_out);
    LAUNCHED();
    return BSGD_OK;
}

__global__ void set_step_kernel(int64_t *ctl, double *xpart, double *scal, const double *stats, double tv,
                                double iters, double restarts, double conv, double fell) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) xpart[k] = stats[k];
        ctl[0] = 1;
        scal[0] = tv; scal[1] = iters; scal[2] = restarts; scal[3] = conv; scal[4] = fell;
    }
}

__global__ void set_step_ctl_kernel(int64_t *ctl, double *xpart, double *scal, const double *stats, const FgpCtl *c) {
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) xpart[k] = stats[k];
        ctl[0] = 1;
        scal[0] = c->fell ? c->tv_b : c->tv_out;
        scal[1] = c->iters; scal[2] = c->restarts; scal[3] = c->done; scal[4] = c->fell;
    }
}

int bsgd_slab_decide(const bsgd_slab *s, int32_t stage, int32_t iteration, const double *gathered, int32_t world,
                     const int32_t *program, int32_t nprogram, double tol, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c, stage == 0 || stage == 3 ? true : true);
    if (rc) return rc;
    if (!(s->flags & BSGD_SLAB_DEVICE)) return fail(BSGD_EINVAL, "bsgd_slab_decide needs BSGD_SLAB_DEVICE");
    if (!gathered || !program) return fail(BSGD_EINVAL, "gathered and program are required");
    if (world < 1 || world > kSlabRanks || nprogram < 1 || nprogram > kSlabProgram)
        return fail(BSGD_EINVAL, "slab program: %d ranks, %d ops (at most %d ranks)", world, nprogram, kSlabRanks);
    if (stage < 0 || stage > 3) return fail(BSGD_EINVAL, "stage must be 0..3");
    SlabProgram prog = {};
    prog.n = nprogram;
    int depth = 0;
    for (int i = 0; i < nprogram; ++i) {
        if (program[i] >= world || program[i] < -1) return fail(BSGD_EINVAL, "bad slab program op %d", program[i]);
        prog.op[i] = (int8_t)program[i];
        depth += program[i] >= 0 ? 1 : -1;
        if (depth < 1 || depth > kSlabRanks) return fail(BSGD_EINVAL, "slab program is not a valid postfix sum");
    }
    if (depth != 1) return fail(BSGD_EINVAL, "slab program leaves %d values", depth);
    c.v.a.tol = tol;
    cudaStream_t st = (cudaStream_t)stream;
    const bool sum2 = stage == 0 || stage == 3;
    if (c.dim == 3) {
        if (sum2) slab_decide_kernel<3, 2><<<1, 32, 0, st>>>(c.v, stage, iteration, gathered, prog);
        else slab_decide_kernel<3, 7><<<1, 32, 0, st>>>(c.v, stage, iteration, gathered, prog);
    } else {
        if (sum2) slab_decide_kernel<2, 2><<<1, 32, 0, st>>>(c.v, stage, iteration, gathered, prog);
        else slab_decide_kernel<2, 5><<<1, 32, 0, st>>>(c.v, stage, iteration, gathered, prog);
    }
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_slab_set_step(const bsgd_slab *s, int64_t cols, const bsgd_epoch_args *a, const double *stats_dev,
                       void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c, false);
    if (rc) return rc;
    if (!(s->flags & BSGD_SLAB_DEVICE)) return fail(BSGD_EINVAL, "bsgd_slab_set_step needs BSGD_SLAB_DEVICE");
    Ws ws;
    rc = check_epoch_args(cols, a, &ws);
    if (rc) return rc;
    if (!stats_dev) return fail(BSGD_EINVAL, "stats_dev is NULL");
    set_step_ctl_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ws.ctl, ws.xpart, ws.scal, stats_dev, c.v.ctl);
    LAUNCHED();
    return BSGD_OK;
}

int bsgd_slab_info(const bsgd_slab *s, int32_t *info_out, double *tv_out, void *stream) {
    SlabCtx c;
    int rc = slab_ctx(s, c, false);
    if (rc) return rc;
    if (!(s->flags & BSGD_SLAB_DEVICE)) return fail(BSGD_EINVAL, "bsgd_slab_info needs BSGD_SLAB_DEVICE");
    if (!info_out) return fail(BSGD_EINVAL, "info_out is NULL");
    FgpCtl h;
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaMemcpyAsync(&h, c.v.ctl, sizeof(FgpCtl), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    info_out[0] = h.iters; info_out[1] = h.done; info_out[2] = h.restarts; info_out[3] = h.fell;
    if (tv_out) *tv_out = h.fell ? h.tv_b : h.tv_out;
    return BSGD_OK;
}

int bsgd_epoch_set_step(int64_t cols, const bsgd_epoch_args *a, const double *stats_dev, double tv,
                        int32_t iterations, int32_t restarts, int32_t converged, int32_t fell_back, void *stream) {
    Ws ws;
    int rc = check_epoch_args(cols, a, &ws);
    if (rc) return rc;
    if (!stats_dev) return fail(BSGD_EINVAL, "stats_dev is NULL");
    set_step_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ws.ctl, ws.xpart, ws.scal, stats_dev, tv, iterations,
                                                        restarts, converged, fell_back);
    LAUNCHED();
    return BSGD_OK;
}

}  // extern "C"
