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

// DB: two windows, and while the CTA computes tile i from one, cp.async gathers
// tile i + gridDim.x's distinct columns into the other (used when two windows
// still leave room for several CTAs per SM; otherwise one window and the
// overlap comes from the other resident CTAs).
template <typename V, bool DB, class Epi>
__global__ void __launch_bounds__(kThreads) gtile_kernel(GTiles T, const double *__restrict__ vec, Epi epi,
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
            for (int j = threadIdx.x; j < nu; j += kThreads) gt_cp_async8(w + j, vec + __ldg(T.uni + u0 + j));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int b = 0;
    if constexpr (DB) gather(blockIdx.x, win);
    for (int64_t t = blockIdx.x; t < T.ntiles; t += gridDim.x) {
        double *w = win + (size_t)b * T.max_union;
        if constexpr (DB) {
            gather(t + gridDim.x, win + (size_t)(b ^ 1) * T.max_union);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            gather(t, win);
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int64_t r0 = T.tile_ptr[t], nr = T.tile_ptr[t + 1] - r0;
        double s = 0.0;
        int64_t row = -1;
        if (tr < nr) {
            row = T.tile_rows[r0 + tr];
            const int64_t beg = T.row_ptr[r0 + tr], end = T.row_ptr[r0 + tr + 1];
            int64_t k = beg + gl;
            for (; k + 48 < end; k += 64) {
                const uint16_t l0 = __ldg(T.loc + k), l1 = __ldg(T.loc + k + 16);
                const uint16_t l2 = __ldg(T.loc + k + 32), l3 = __ldg(T.loc + k + 48);
                const V v0 = ld_stream(val + k, pol), v1 = ld_stream(val + k + 16, pol);
                const V v2 = ld_stream(val + k + 32, pol), v3 = ld_stream(val + k + 48, pol);
                s = fma((double)v0, w[l0], s);
                s = fma((double)v1, w[l1], s);
                s = fma((double)v2, w[l2], s);
                s = fma((double)v3, w[l3], s);
            }
            for (; k < end; k += 16) s = fma((double)ld_stream(val + k, pol), w[__ldg(T.loc + k)], s);
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
