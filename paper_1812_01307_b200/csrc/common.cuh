// Shared device helpers for the BSGD-TV sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bsgd {

constexpr int kThreads = 256;           // threads per CTA for every streaming kernel
constexpr int kMaxPartials = 4096;      // upper bound on CTAs that write a reduction partial
constexpr int kNumSMs = 148;            // B200

// ---- IEEE ops without contraction: the reference evaluates every product and
// sum with its own rounding (numpy / scipy, no FMA), and the TV prox mirrors
// that elementwise so its restart / stop decisions see the same values.
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }

// ---- streaming loads: the A / A^T value and index streams are touched once per
// product, so they bypass L1 and are marked evict-first in L2, which keeps the
// gathered x / r vectors (a few MB) resident in the 126 MB L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ int32_t ld_stream(const int32_t *p, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream(const float *p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ int4 ld_stream4(const int32_t *p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 ld_stream4(const float *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ double2 ld_stream2(const double *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

// ---- deterministic reductions: fixed shuffle tree, fixed warp order.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Sum K values over the CTA; every thread receives the totals. `sm` must hold
// K * (blockDim.x / 32) doubles.  Ends with a __syncthreads().
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double *sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) sm[k * nw + warp] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += sm[k * nw + w];
        v[k] = s;
    }
    __syncthreads();
}

// Sum `n` per-CTA partials laid out as part[b * K + k] in a fixed order,
// executed by one full warp (all 32 lanes get the totals).
template <int K>
__device__ __forceinline__ void warp_sum_partials(const double *part, int n, double (&out)[K]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int b = lane; b < n; b += 32) s += part[(size_t)b * K + k];
        out[k] = warp_sum(s);
    }
}

}  // namespace bsgd
