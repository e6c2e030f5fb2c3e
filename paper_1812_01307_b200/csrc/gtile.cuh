// Gather-tiled CSR products for matrices whose rows come in groups that share
// columns (parallel-beam CT: 4x4 pixel tiles of A^T share 4.0 entries per
// distinct ray, 4 angles x 4 bins of A share 3.45 entries per distinct pixel).
//
// The CSR kernel (spmv.cuh) gathers one vector element per nonzero and is
// bounded by the L1 tag stage at ~1 distinct sector per SM per cycle
// (profiles/r01_gather_microbench.md).  Here a CTA takes one tile of <= 16
// rows: it gathers the tile's distinct columns once into shared memory (the
// plan stores each tile's sorted column union and, per entry, its position in
// it as uint16), then 16 lanes per row stream the row's (position, value)
// pairs and read the vector from shared memory (~5 loads/SM/cycle).  Global
// gathers drop by the tile's reuse factor.  Per-row arithmetic is the CSR
// kernel's G = 16 form: lane-strided float64 partial sums and a fixed
// shuffle tree, deterministic run to run.
//
// Stream layout: each row is padded (position 0, value 0) to whole blocks of
// 128 entries, and inside a block entry e = 16 m + l is stored at 8 l + m, so
// lane l fetches its eight lane-strided entries l, l + 16, ..., l + 112 with one
// 16-byte position load and 16-byte value loads.  The stream loads were the
// kernel's latency wall (profiles/r01_ct_spmv.md: the shared-memory address
// computations waited on 2-byte position loads); the summation order is the
// lane-strided order of the unblocked form.
#pragma once

#include "common.cuh"

namespace bsgd {

struct GTiles {
    int64_t ntiles;
    const int64_t *tile_ptr;   // [ntiles + 1] -> tile rows
    const int32_t *tile_rows;  // row id of each tile row
    const int64_t *row_ptr;    // [tile rows + 1] entries in tile-row order
    const uint16_t *loc;       // entry -> position in the tile's column union
    const void *val;           // entry values (V)
    const int64_t *uni_ptr;    // [ntiles + 1]
    const int32_t *uni;        // sorted distinct columns per tile
    int max_union;             // largest union (shared-memory window in doubles)
};

constexpr int kGTileRows = 16;

__device__ __forceinline__ void gt_cp_async8(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}

constexpr int kGTileBlock = 128;   // stream block (entries) of one 16-lane row group

// eight consecutive stored values of a block as float64
__device__ __forceinline__ void gt_load8(const float *p, double (&v)[8], uint64_t pol) {
    const float4 a = ld_stream4(p, pol), b = ld_stream4(p + 4, pol);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void gt_load8(const double *p, double (&v)[8], uint64_t pol) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double2 a = ld_stream2(p + 2 * q, pol);
        v[2 * q] = a.x;
        v[2 * q + 1] = a.y;
    }
}

// one stream block of a lane: eight packed positions and the raw values
template <typename V>
struct GtBlk {
    int4 l;
    V v[8];
};

template <typename V>
__device__ __forceinline__ void gt_load_blk(const uint16_t *loc, const V *val, int64_t k, GtBlk<V> &b,
                                            uint64_t pol) {
    b.l = ld_stream4(reinterpret_cast<const int32_t *>(loc + k), pol);
    if constexpr (sizeof(V) == 4) {
        const float4 x = ld_stream4(val + k, pol), y = ld_stream4(val + k + 4, pol);
        b.v[0] = x.x; b.v[1] = x.y; b.v[2] = x.z; b.v[3] = x.w; b.v[4] = y.x; b.v[5] = y.y; b.v[6] = y.z; b.v[7] = y.w;
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 x = ld_stream2(val + k + 2 * q, pol);
            b.v[2 * q] = x.x;
            b.v[2 * q + 1] = x.y;
        }
    }
}

template <typename V>
__device__ __forceinline__ double gt_use_blk(const GtBlk<V> &b, const double *w, double s) {
    const uint32_t q[4] = {(uint32_t)b.l.x, (uint32_t)b.l.y, (uint32_t)b.l.z, (uint32_t)b.l.w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        s = fma((double)b.v[2 * m], w[q[m] & 0xFFFFu], s);
        s = fma((double)b.v[2 * m + 1], w[q[m] >> 16], s);
    }
    return s;
}

// s += v[m] * w[pos[m]] for the eight packed uint16 positions, in order m = 0..7
__device__ __forceinline__ double gt_fma8(const int4 l, const double (&v)[8], const double *w, double s) {
    const uint32_t q[4] = {(uint32_t)l.x, (uint32_t)l.y, (uint32_t)l.z, (uint32_t)l.w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        s = fma(v[2 * m], w[q[m] & 0xFFFFu], s);
        s = fma(v[2 * m + 1], w[q[m] >> 16], s);
    }
    return s;
}

// DB: two windows, and while the CTA computes tile i from one, cp.async gathers
// tile i + gridDim.x's distinct columns into the other (used when two windows
// still leave room for several CTAs per SM; otherwise one window and the
// overlap comes from the other resident CTAs).
template <typename V, bool DB, class Epi>
__global__ void __launch_bounds__(kThreads, 3) gtile_kernel(GTiles T, const double *__restrict__ vec, Epi epi,
                                                         double *part, int64_t *cnt) {
    extern __shared__ double win[];   // [DB ? 2 : 1][max_union]
    __shared__ double sm[8 * (kThreads / 32)];
    const int lane = threadIdx.x & 31;
    const int tr = threadIdx.x >> 4;   // tile row (two per warp)
    const int gl = threadIdx.x & 15;   // lane within the row
    const unsigned gmask = 0xFFFFu << (lane & 16);
    const uint64_t pol = policy_evict_first();
    const V *__restrict__ val = reinterpret_cast<const V *>(T.val);
    auto gather = [&](int64_t t, double *w) {
        if (t < T.ntiles) {
            const int64_t u0 = T.uni_ptr[t];
            const int nu = (int)(T.uni_ptr[t + 1] - u0);
            // four union ids loaded before their copies are issued
            int j = threadIdx.x;
            for (; j + 3 * kThreads < nu; j += 4 * kThreads) {
                int32_t c[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) c[q] = __ldg(T.uni + u0 + j + q * kThreads);
#pragma unroll
                for (int q = 0; q < 4; ++q) gt_cp_async8(w + j + q * kThreads, vec + c[q]);
            }
            for (; j < nu; j += kThreads) gt_cp_async8(w + j, vec + __ldg(T.uni + u0 + j));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int b = 0;
    if constexpr (DB) gather(blockIdx.x, win);
    for (int64_t t = blockIdx.x; t < T.ntiles; t += gridDim.x) {
        double *w = win + (size_t)b * T.max_union;
        if constexpr (DB) gather(t + gridDim.x, win + (size_t)(b ^ 1) * T.max_union);
        else gather(t, win);
        // the row's first two stream blocks are fetched while the union lands
        const int64_t r0 = T.tile_ptr[t], nr = T.tile_ptr[t + 1] - r0;
        int64_t row = -1, k = 0, end = 0;
        GtBlk<V> c0, c1, n0, n1;
        if (tr < nr) {
            row = T.tile_rows[r0 + tr];
            k = T.row_ptr[r0 + tr] + 8 * gl;
            end = T.row_ptr[r0 + tr + 1];   // multiples of 128
            if (k < end) gt_load_blk(T.loc, val, k, c0, pol);
            if (k + 128 < end) gt_load_blk(T.loc, val, k + 128, c1, pol);
        }
        if constexpr (DB) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        double s = 0.0;
        // software pipeline: the next two blocks are in flight while two are summed
        for (; k < end; k += 256) {
            if (k + 256 < end) gt_load_blk(T.loc, val, k + 256, n0, pol);
            if (k + 384 < end) gt_load_blk(T.loc, val, k + 384, n1, pol);
            s = gt_use_blk(c0, w, s);
            if (k + 128 < end) s = gt_use_blk(c1, w, s);
            c0 = n0;
            c1 = n1;
        }
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(gmask, s, off, 16);
        if (gl == 0 && row >= 0) epi(row, s);
        __syncthreads();  // the window is refilled (DB: two tiles later)
        if constexpr (DB) b ^= 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.flush(v);
        block_sum<Epi::K>(v, sm);
        if (threadIdx.x == 0 && part != nullptr)
            for (int q = 0; q < Epi::K; ++q) part[(size_t)blockIdx.x * Epi::K + q] = v[q];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != nullptr) cnt[0] = gridDim.x;
}

}  // namespace bsgd
