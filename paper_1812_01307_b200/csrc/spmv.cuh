// CSR row-product kernels for the two SpMV directions of a BSGD-TV epoch.
//
// K1 (forward)    : r[row] = y[row] - sum_k A[row, k] x[k]       on A   (CSR)
// K2 (transposed) : g[col] = 2 sum_k A[k, col] r[k]  (+ step)     on A^T (CSR)
// Both are the same row-product over a CSR stream with a fused epilogue.
//
// Mapping: a warp owns 32/G consecutive rows per pass, G lanes per row
// (G = 4 for rows under 48 nonzeros such as the 32-nnz random system, 8 under
// 256, 32 for CT rays of ~400-1800).  Each lane streams a strided slice of its row's (index,
// value) pairs with L1-bypassing evict-first loads, gathers the vector
// through the read-only path (the vector stays L2-resident), and accumulates
// in float64.  The in-row reduction is a fixed shuffle tree, so results are
// deterministic run to run.
#pragma once

#include "common.cuh"

namespace bsgd {

// ---------------------------------------------------------------------------
// epilogues: called once per row by the row's lane 0 with the float64 sum
// ---------------------------------------------------------------------------

struct EpiStore {  // out[row] = scale * s  (matvec / rmatvec: 1; partial gradient: 2, exact)
    double *out;
    double scale;
    static constexpr int K = 0;
    __device__ __forceinline__ void operator()(int64_t row, double s) { out[row] = scale * s; }
    __device__ __forceinline__ void flush(double *) {}
};

struct EpiResid {  // r[row] = y[row] - s, accumulate ||r||^2  (assemble_residual, blockops.py:264-278)
    const double *y;
    double *r;
    double acc = 0.0;
    static constexpr int K = 1;
    __device__ __forceinline__ void operator()(int64_t row, double s) {
        const double v = rn_sub(y[row], s);
        r[row] = v;
        acc += v * v;
    }
    __device__ __forceinline__ void flush(double *v) { v[0] = acc; }
};

// g = 2 * s (solvers.py:299-303), x_new = x_k + mu * g (solvers.py:308).
// With a prox the step is scattered into image order (tv.py:87-93) for the
// FGP kernel; without one it is the iterate, and its epoch statistics
// (||x||^2, ||x - x_true||^2, (x_new - x_k).g, ||x_new - x_k||^2) are fused.
struct EpiStep {
    double *g;
    const double *xk;
    double mu;
    double *xn;            // lam == 0: iterate out
    double *uimg;          // lam > 0: image-order step out
    const int64_t *perm;   // NULL = identity
    const double *xtrue;   // NULL = no relative error
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    static constexpr int K = 4;
    __device__ __forceinline__ void operator()(int64_t col, double s) {
        const double gg = 2.0 * s;
        g[col] = gg;
        const double xo = xk[col];
        const double xv = rn_add(xo, rn_mul(mu, gg));
        if (uimg != nullptr) {
            uimg[perm != nullptr ? perm[col] : col] = xv;
        } else {
            xn[col] = xv;
            const double d = rn_sub(xv, xo);
            acc[0] += xv * xv;
            if (xtrue != nullptr) {
                const double e = xv - xtrue[col];
                acc[1] += e * e;
            }
            acc[2] += d * gg;
            acc[3] += d * d;
        }
    }
    __device__ __forceinline__ void flush(double *v) {
        v[0] = acc[0]; v[1] = acc[1]; v[2] = acc[2]; v[3] = acc[3];
    }
};

// The step with the TV prox on (lam > 0): g = 2 s and the prox input b = x_k + mu g
// scattered to image order; no statistics (the prox's output pass computes them
// from x_next), so no accumulators and no partials -- the K2 kernels keep fewer
// live registers (gtile_kernel<float, *, EpiStep> spilled 60-64 B at its
// 80-register cap).
struct EpiStepImg {
    double *g;
    const double *xk;
    double mu;
    double *uimg;
    const int64_t *perm;   // NULL = identity
    static constexpr int K = 0;
    __device__ __forceinline__ void operator()(int64_t col, double s) {
        const double gg = 2.0 * s;
        g[col] = gg;
        uimg[perm != nullptr ? perm[col] : col] = rn_add(xk[col], rn_mul(mu, gg));
    }
    __device__ __forceinline__ void flush(double *) {}
};

struct EpiNone {
    static constexpr int K = 0;
    __device__ __forceinline__ void operator()(int64_t, double) {}
    __device__ __forceinline__ void flush(double *) {}
};

// ---------------------------------------------------------------------------
// one CSR operand (matrix + gathered vector)
// ---------------------------------------------------------------------------
template <typename V>
struct Csr {
    int64_t nrows;
    const int64_t *ptr;
    const int32_t *idx;
    const V *val;
    const double *vec;
};

template <typename V, int G, class Epi>
__device__ __forceinline__ void csr_rows(const Csr<V> &A, int64_t warp_id, int64_t nwarps, Epi &epi) {
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int sub = lane / G;
    const int gl = lane % G;
    const uint64_t pol = policy_evict_first();
    const int32_t *__restrict__ idx = A.idx;
    const V *__restrict__ val = A.val;
    const double *__restrict__ vec = A.vec;
    for (int64_t base = warp_id * RPW; base < A.nrows; base += nwarps * RPW) {
        const int64_t row = base + sub;
        double s = 0.0;
        if (row < A.nrows) {
            const int64_t beg = A.ptr[row];
            const int64_t end = A.ptr[row + 1];
            if constexpr (sizeof(V) == 4 && G <= 8) {
                // short rows: 16-byte streaming loads over the 4-aligned body of the row:
                // one L1 request moves 4 (index, value) pairs, leaving the L1 tag stage to
                // the random gathers (profiles/r01_spmv_baseline.md).  Used with G = 4 / 8
                // (8-16 entries per lane); with 32 lanes on 128-nnz rows it measured +4%
                const int64_t b4 = (beg + 3) & ~(int64_t)3;
                const int64_t e4 = end & ~(int64_t)3;
                if (b4 < e4) {
                    for (int64_t k = beg + gl; k < b4; k += G)
                        s = fma((double)ld_stream(val + k, pol), __ldg(vec + ld_stream(idx + k, pol)), s);
                    int64_t k = b4 + 4 * gl;
                    for (; k + 4 * G < e4; k += 8 * G) {
                        const int4 c0 = ld_stream4(idx + k, pol);
                        const int4 c1 = ld_stream4(idx + k + 4 * G, pol);
                        const float4 v0 = ld_stream4(reinterpret_cast<const float *>(val) + k, pol);
                        const float4 v1 = ld_stream4(reinterpret_cast<const float *>(val) + k + 4 * G, pol);
                        const double x0 = __ldg(vec + c0.x), x1 = __ldg(vec + c0.y), x2 = __ldg(vec + c0.z),
                                     x3 = __ldg(vec + c0.w), x4 = __ldg(vec + c1.x), x5 = __ldg(vec + c1.y),
                                     x6 = __ldg(vec + c1.z), x7 = __ldg(vec + c1.w);
                        s = fma((double)v0.x, x0, s); s = fma((double)v0.y, x1, s);
                        s = fma((double)v0.z, x2, s); s = fma((double)v0.w, x3, s);
                        s = fma((double)v1.x, x4, s); s = fma((double)v1.y, x5, s);
                        s = fma((double)v1.z, x6, s); s = fma((double)v1.w, x7, s);
                    }
                    for (; k < e4; k += 4 * G) {
                        const int4 c0 = ld_stream4(idx + k, pol);
                        const float4 v0 = ld_stream4(reinterpret_cast<const float *>(val) + k, pol);
                        const double x0 = __ldg(vec + c0.x), x1 = __ldg(vec + c0.y), x2 = __ldg(vec + c0.z),
                                     x3 = __ldg(vec + c0.w);
                        s = fma((double)v0.x, x0, s); s = fma((double)v0.y, x1, s);
                        s = fma((double)v0.z, x2, s); s = fma((double)v0.w, x3, s);
                    }
                    for (int64_t t = e4 + gl; t < end; t += G)
                        s = fma((double)ld_stream(val + t, pol), __ldg(vec + ld_stream(idx + t, pol)), s);
                } else {
                    for (int64_t t = beg + gl; t < end; t += G)
                        s = fma((double)ld_stream(val + t, pol), __ldg(vec + ld_stream(idx + t, pol)), s);
                }
            } else {
                int64_t k = beg + gl;
                for (; k + 3 * G < end; k += 4 * G) {
                    const int32_t c0 = ld_stream(idx + k, pol);
                    const int32_t c1 = ld_stream(idx + k + G, pol);
                    const int32_t c2 = ld_stream(idx + k + 2 * G, pol);
                    const int32_t c3 = ld_stream(idx + k + 3 * G, pol);
                    const V v0 = ld_stream(val + k, pol);
                    const V v1 = ld_stream(val + k + G, pol);
                    const V v2 = ld_stream(val + k + 2 * G, pol);
                    const V v3 = ld_stream(val + k + 3 * G, pol);
                    const double x0 = __ldg(vec + c0);
                    const double x1 = __ldg(vec + c1);
                    const double x2 = __ldg(vec + c2);
                    const double x3 = __ldg(vec + c3);
                    s = fma((double)v0, x0, s);
                    s = fma((double)v1, x1, s);
                    s = fma((double)v2, x2, s);
                    s = fma((double)v3, x3, s);
                }
                for (; k < end; k += G) {
                    const int32_t c0 = ld_stream(idx + k, pol);
                    const V v0 = ld_stream(val + k, pol);
                    s = fma((double)v0, __ldg(vec + c0), s);
                }
            }
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (gl == 0 && row < A.nrows) epi(row, s);
    }
}

// Two independent CSR products in one grid: CTAs [0, nblkA) run part A, the
// rest run part B (used to overlap K1(x_k) and K2(r_k), which read the same
// snapshot, solvers.py:276-290).  Each part writes one partial per CTA.
template <typename V, int GA, int GB, class EA, class EB>
__global__ void __launch_bounds__(kThreads) dual_csr_kernel(Csr<V> A, EA ea, double *partA, int nblkA,
                                                            int64_t *cntA, Csr<V> B, EB eb,
                                                            double *partB, int64_t *cntB) {
    __shared__ double sm[8 * (kThreads / 32)];
    const int wpb = kThreads / 32;
    if ((int)blockIdx.x < nblkA) {
        const int64_t warp = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
        csr_rows<V, GA>(A, warp, (int64_t)nblkA * wpb, ea);
        if constexpr (EA::K > 0) {
            double v[EA::K];
            ea.flush(v);
            block_sum<EA::K>(v, sm);
            if (threadIdx.x == 0 && partA != nullptr)
                for (int k = 0; k < EA::K; ++k) partA[(size_t)blockIdx.x * EA::K + k] = v[k];
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && cntA != nullptr) cntA[0] = nblkA;
    } else {
        const int nblkB = gridDim.x - nblkA;
        const int bb = blockIdx.x - nblkA;
        const int64_t warp = (int64_t)bb * wpb + (threadIdx.x >> 5);
        csr_rows<V, GB>(B, warp, (int64_t)nblkB * wpb, eb);
        if constexpr (EB::K > 0) {
            double v[EB::K];
            eb.flush(v);
            block_sum<EB::K>(v, sm);
            if (threadIdx.x == 0 && partB != nullptr)
                for (int k = 0; k < EB::K; ++k) partB[(size_t)bb * EB::K + k] = v[k];
        }
        if (bb == 0 && threadIdx.x == 0 && cntB != nullptr) cntB[0] = nblkB;
    }
}

// ---------------------------------------------------------------------------
// blocked stream (long rows): GB lanes per row, each row padded to whole blocks
// of 4 GB entries, entry GB m + l of a block stored at 4 l + m, so lane l
// fetches its four lane-strided entries l, l + GB, l + 2 GB, l + 3 GB with one
// 16-byte index load and one 16-byte value load (float32; two for float64), two
// blocks in flight; padding entries repeat the row's last column with value 0.
// The unblocked G = 32 loop stalls on its 4-byte index loads before it can form
// the gather addresses (profiles/r01_ct_spmv.md).  With GB = 32 the per-lane
// order is the unblocked kernel's (bit-identical); the plan uses GB = 4 / 8 so
// that one warp covers 8 / 4 adjacent rays, whose gathers share sectors inside
// one instruction (tomographic rays of neighbouring bins).
// ---------------------------------------------------------------------------
// lanes per row of the blocked kernel: GB lanes, blocks of 4 GB entries
template <typename V>
struct CsrB {
    int64_t nrows;
    const int64_t *ptr;   // [nrows + 1], multiples of the block (4 GB entries)
    const int32_t *idx;
    const V *val;
    const double *vec;
    // compressed indices (CMP): 16-bit offsets from two bases per block, half[b] = (least
    // column of the block's first 2 GB entries, of its last 2 GB): a lane's entries
    // l, l + GB come from the first half and l + 2 GB, l + 3 GB from the second, so
    // column = base + offset with no dependent chain; 2 + 8 / (4 GB) bytes per entry
    const int2 *half = nullptr;
    const uint16_t *off = nullptr;
};

__device__ __forceinline__ uint2 ld_stream_u2(const void *p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ int2 ld_stream_i2(const int2 *p, uint64_t pol) {
    int2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

// the lane's four columns of the block at entry k (k = block start + 4 lane)
template <bool CMP, int GB, typename V>
__device__ __forceinline__ int4 blk_cols(const CsrB<V> &A, int64_t k, uint64_t pol) {
    if constexpr (CMP) {
        const int2 h = ld_stream_i2(A.half + k / (4 * GB), pol);
        const uint2 d = ld_stream_u2(A.off + k, pol);
        return make_int4(h.x + (int32_t)(d.x & 0xFFFFu), h.x + (int32_t)(d.x >> 16), h.y + (int32_t)(d.y & 0xFFFFu),
                         h.y + (int32_t)(d.y >> 16));
    } else {
        return ld_stream4(A.idx + k, pol);
    }
}

__device__ __forceinline__ void blk_vals(const float *p, double (&v)[4], uint64_t pol) {
    const float4 a = ld_stream4(p, pol);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void blk_vals(const double *p, double (&v)[4], uint64_t pol) {
    const double2 a = ld_stream2(p, pol), b = ld_stream2(p + 2, pol);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

template <typename V, int GB, class Epi, bool CMP>
__device__ __forceinline__ void csr_blocked_body(const CsrB<V> &A, Epi &epi, double *part, int64_t *cnt) {
    constexpr int BLK = 4 * GB;
    constexpr int RPW = 32 / GB;
    __shared__ double sm[8 * (kThreads / 32)];
    const int lane = threadIdx.x & 31;
    const int sub = lane / GB, gl = lane % GB;
    const uint64_t pol = policy_evict_first();
    const double *__restrict__ vec = A.vec;
    const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t base = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * RPW; base < A.nrows;
         base += nw * RPW) {
        const int64_t row = base + sub;
        double s = 0.0;
        if (row < A.nrows) {
            const int64_t beg = A.ptr[row], end = A.ptr[row + 1];
            int64_t k = beg + 4 * gl;
            for (; k + BLK < end; k += 2 * BLK) {
                const int4 ca = blk_cols<CMP, GB>(A, k, pol), cb = blk_cols<CMP, GB>(A, k + BLK, pol);
                double va[4], vb[4];
                blk_vals(A.val + k, va, pol);
                blk_vals(A.val + k + BLK, vb, pol);
                const double xa0 = __ldg(vec + ca.x), xa1 = __ldg(vec + ca.y), xa2 = __ldg(vec + ca.z),
                             xa3 = __ldg(vec + ca.w), xb0 = __ldg(vec + cb.x), xb1 = __ldg(vec + cb.y),
                             xb2 = __ldg(vec + cb.z), xb3 = __ldg(vec + cb.w);
                s = fma(va[0], xa0, s); s = fma(va[1], xa1, s); s = fma(va[2], xa2, s); s = fma(va[3], xa3, s);
                s = fma(vb[0], xb0, s); s = fma(vb[1], xb1, s); s = fma(vb[2], xb2, s); s = fma(vb[3], xb3, s);
            }
            if (k < end) {
                const int4 ca = blk_cols<CMP, GB>(A, k, pol);
                double va[4];
                blk_vals(A.val + k, va, pol);
                const double xa0 = __ldg(vec + ca.x), xa1 = __ldg(vec + ca.y), xa2 = __ldg(vec + ca.z),
                             xa3 = __ldg(vec + ca.w);
                s = fma(va[0], xa0, s); s = fma(va[1], xa1, s); s = fma(va[2], xa2, s); s = fma(va[3], xa3, s);
            }
        }
#pragma unroll
        for (int off = GB / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (gl == 0 && row < A.nrows) epi(row, s);
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.flush(v);
        block_sum<Epi::K>(v, sm);
        if (threadIdx.x == 0 && part != nullptr)
            for (int q = 0; q < Epi::K; ++q) part[(size_t)blockIdx.x * Epi::K + q] = v[q];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != nullptr) cnt[0] = gridDim.x;
}

// Two register budgets of the same body: ptxas fits the loop in 40 registers (48 warps
// per SM) when left alone and in 32 (64 warps) when asked for 8 CTAs per SM, both
// without spills (any other explicit bound measured slower: 1 -> 64 registers, 6 -> a
// different 40-register schedule).  Which one wins depends on the product (launch_blocked).
template <typename V, int GB, class Epi, bool CMP = false>
__global__ void __launch_bounds__(kThreads) csr_blocked_kernel(CsrB<V> A, Epi epi, double *part, int64_t *cnt) {
    csr_blocked_body<V, GB, Epi, CMP>(A, epi, part, cnt);
}
template <typename V, int GB, class Epi, bool CMP = false>
__global__ void __launch_bounds__(kThreads, 8) csr_blocked_w64_kernel(CsrB<V> A, Epi epi, double *part,
                                                                      int64_t *cnt) {
    csr_blocked_body<V, GB, Epi, CMP>(A, epi, part, cnt);
}

// compress the blocked indices (CsrB::half / off): one thread per block of 4 gb stored
// entries (stored position 4 l + m holds entry gb m + l, so m < 2 is the first half);
// *bad != 0 when an offset does not fit 16 bits
__global__ void blk_compress_kernel(int64_t nblocks, int gb, const int32_t *idx, int2 *half, uint16_t *off, int *bad) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int4 *c = reinterpret_cast<const int4 *>(idx) + b * gb;
        int32_t lo0 = INT32_MAX, lo1 = INT32_MAX;
        for (int l = 0; l < gb; ++l) {
            const int4 v = c[l];
            lo0 = min(lo0, min(v.x, v.y));
            lo1 = min(lo1, min(v.z, v.w));
        }
        half[b] = make_int2(lo0, lo1);
        bool over = false;
        for (int l = 0; l < gb; ++l) {
            const int4 v = c[l];
            const int64_t d0 = (int64_t)v.x - lo0, d1 = (int64_t)v.y - lo0, d2 = (int64_t)v.z - lo1,
                          d3 = (int64_t)v.w - lo1;
            over |= d0 > 65535 || d1 > 65535 || d2 > 65535 || d3 > 65535;
            ushort4 o;
            o.x = (uint16_t)d0; o.y = (uint16_t)d1; o.z = (uint16_t)d2; o.w = (uint16_t)d3;
            reinterpret_cast<ushort4 *>(off)[b * gb + l] = o;
        }
        if (over) atomicExch(bad, 1);
    }
}

// Order of the blocked stream's gathers over the vector's grid (rows of n columns,
// element c row-major): order 1 = 4 x 4 tiles (one 128-byte line each; a ragged last
// tile column / row is padded), 4 = 8 x 2 tiles (8 grid rows x 2 columns), 5 = 2 x 8
// tiles, 2 = Morton (Z) order (square power-of-two grids)
__device__ __forceinline__ uint32_t spread_bits16(uint32_t v) {
    v &= 0xffffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__device__ __forceinline__ int32_t blk_order_map(int32_t c, int n, int order) {
    const int y = c / n, x = c - y * n;
    if (order == 1) return ((y >> 2) * ((n + 3) >> 2) + (x >> 2)) * 16 + ((y & 3) << 2) + (x & 3);
    if (order == 4) return ((y >> 3) * ((n + 1) >> 1) + (x >> 1)) * 16 + ((y & 7) << 1) + (x & 1);   // 8 x 2 tiles
    if (order == 5) return ((y >> 1) * ((n + 7) >> 3) + (x >> 3)) * 16 + ((y & 1) << 3) + (x & 7);   // 2 x 8 tiles
    return (int32_t)((spread_bits16((uint32_t)y) << 1) | spread_bits16((uint32_t)x));
}
__global__ void blk_renumber_kernel(int64_t total, int32_t *idx, int n, int order) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        idx[i] = blk_order_map(idx[i], n, order);
}
__global__ void blk_permute_kernel(int64_t cols, const double *x, double *xt, int n, int order) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x)
        xt[blk_order_map((int32_t)c, n, order)] = x[c];
}

// Footprint of a gather instruction on the grid: over every run of 16 consecutive
// entries of a row, the spans (max - min + 1) of their grid rows and grid columns,
// summed into acc[0] / acc[1] (acc[2] counts the runs).  One warp per row.
__global__ void blk_span_kernel(int64_t nrows, const int64_t *ptr, const int32_t *idx, int gw,
                                unsigned long long *acc) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long sy = 0, sx = 0, cnt = 0;
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrows; r += nw) {
        const int64_t beg = ptr[r], end = ptr[r + 1];
        for (int64_t k = beg + 16 * lane; k + 16 <= end; k += 16 * 32) {
            int y0 = INT32_MAX, y1 = -1, x0 = INT32_MAX, x1 = -1;
            for (int q = 0; q < 16; ++q) {
                const int c = idx[k + q];
                const int y = c / gw, x = c - y * gw;
                y0 = min(y0, y); y1 = max(y1, y); x0 = min(x0, x); x1 = max(x1, x);
            }
            sy += (unsigned long long)(y1 - y0 + 1);
            sx += (unsigned long long)(x1 - x0 + 1);
            ++cnt;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0 && cnt) {
        atomicAdd(acc, sy);
        atomicAdd(acc + 1, sx);
        atomicAdd(acc + 2, cnt);
    }
}

// Histogram of the gaps between consecutive column indices (1 < gap < nbins) over every
// `stride`-th row: a matrix whose gathered vector lives on a row-major grid of width w
// (A^T of a CT system: bins of one angle adjacent, the next angle ~w further) shows a
// sharp peak at ~w.  One warp per sampled row.
__global__ void blk_gap_hist_kernel(int64_t nrows, int64_t stride, const int64_t *ptr, const int32_t *idx,
                                    int nbins, unsigned int *hist) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * stride; r < nrows;
         r += nw * stride) {
        const int64_t beg = ptr[r], end = ptr[r + 1];
        for (int64_t k = beg + lane; k + 1 < end; k += 32) {
            const int64_t d = (int64_t)idx[k + 1] - idx[k];
            if (d > 1 && d < nbins) atomicAdd(hist + d, 1u);
        }
    }
}

// padded row lengths (whole blocks of blk entries) for the blocked copy
__global__ void blk_len_kernel(int64_t rows, const int64_t *ptr, int blk, int64_t *out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        out[r] = (ptr[r + 1] - ptr[r] + blk - 1) / blk * blk;
}

// scatter a canonical CSR into the blocked layout (one warp per row)
template <typename V>
__global__ void __launch_bounds__(kThreads) blk_fill_kernel(int64_t rows, const int64_t *ptr, const int32_t *idx,
                                                            const V *val, const int64_t *bptr, int32_t *bidx,
                                                            V *bval, int gb) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t r = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); r < rows; r += nw) {
        const int64_t beg = ptr[r], len = ptr[r + 1] - beg, ob = bptr[r], plen = bptr[r + 1] - ob;
        const int32_t last = len > 0 ? idx[beg + len - 1] : 0;
        for (int64_t k = lane; k < plen; k += 32) {
            const int64_t e = k % (4 * gb);
            const int64_t o = ob + (k - e) + (e % gb) * 4 + e / gb;
            bidx[o] = k < len ? idx[beg + k] : last;
            bval[o] = k < len ? val[beg + k] : V(0);
        }
    }
}

// ---------------------------------------------------------------------------
// block-restricted products (blockops.py:207-223): rows [r0, r1) of a CSR,
// entries with column in [c0, c1) (a contiguous run: indices are sorted).
// out[row - r0] = sum A[row, c] vec[c - c0].  One warp per row.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *a, int64_t lo, int64_t hi, int64_t key) {
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if ((int64_t)a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <typename V>
__global__ void __launch_bounds__(kThreads) block_seg_kernel(const int64_t *ptr, const int32_t *idx,
                                                             const V *val, int64_t r0, int64_t r1,
                                                             int64_t c0, int64_t c1,
                                                             const double *vec, double *out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t row = r0 + (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < r1; row += nw) {
        int64_t lo = 0, hi = 0;
        if (lane == 0) {
            lo = lower_bound_i32(idx, ptr[row], ptr[row + 1], c0);
            hi = lower_bound_i32(idx, lo, ptr[row + 1], c1);
        }
        lo = __shfl_sync(0xffffffffu, lo, 0);
        hi = __shfl_sync(0xffffffffu, hi, 0);
        double s = 0.0;
        for (int64_t k = lo + lane; k < hi; k += 32) s = fma((double)val[k], vec[idx[k] - c0], s);
        s = warp_sum(s);
        if (lane == 0) out[row - r0] = s;
    }
}

// block-selection bitmask passed by value (up to 256 blocks per side)
struct BlockMask {
    uint64_t w[4];
    __host__ __device__ bool has(int64_t b) const { return (w[b >> 6] >> (b & 63)) & 1ull; }
};

__device__ __forceinline__ int64_t block_of(const int64_t *bounds, int64_t nb, int64_t x) {
    int64_t lo = 0, hi = nb;  // largest b with bounds[b] <= x
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (bounds[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// Stochastic pairs (solvers.py:274-303, alpha/gamma < 1): for rows of the
// selected row blocks, z_cache[j, row] = segment sum over column block j for
// every selected j; then every row's r_next = y - z_cache[0] - ... (ascending j).
template <typename V>
__global__ void __launch_bounds__(kThreads) pair_forward_kernel(const int64_t *ptr, const int32_t *idx,
                                                                const V *val, int64_t rows,
                                                                const int64_t *row_bounds, int64_t M,
                                                                const int64_t *col_bounds, int64_t N,
                                                                BlockMask rsel, BlockMask csel,
                                                                const double *x, const double *y,
                                                                double *z_cache, double *r_next) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t row = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); row < rows; row += nw) {
        if (rsel.has(block_of(row_bounds, M, row))) {
            int64_t lo = ptr[row];
            for (int64_t j = 0; j < N; ++j) {
                int64_t hi = 0;
                if (lane == 0) hi = lower_bound_i32(idx, lo, ptr[row + 1], col_bounds[j + 1]);
                hi = __shfl_sync(0xffffffffu, hi, 0);
                if (csel.has(j)) {
                    double s = 0.0;
                    for (int64_t k = lo + lane; k < hi; k += 32) s = fma((double)val[k], x[idx[k]], s);
                    s = warp_sum(s);
                    if (lane == 0) z_cache[j * rows + row] = s;
                }
                lo = hi;
            }
        }
        __syncwarp();
        if (lane == 0) {
            double acc = y[row];
            for (int64_t j = 0; j < N; ++j) acc = rn_sub(acc, z_cache[j * rows + row]);
            r_next[row] = acc;
        }
    }
}

// g[col] = 2 * sum over selected row blocks (ascending) of the A^T segment sums,
// zero for columns of unselected column blocks (solvers.py:299-303).
template <typename V>
__global__ void __launch_bounds__(kThreads) pair_grad_kernel(const int64_t *tptr, const int32_t *tidx,
                                                             const V *tval, int64_t cols,
                                                             const int64_t *row_bounds, int64_t M,
                                                             const int64_t *col_bounds, int64_t N,
                                                             BlockMask rsel, BlockMask csel,
                                                             const double *r, double *g) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t col = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); col < cols; col += nw) {
        double acc = 0.0;
        if (csel.has(block_of(col_bounds, N, col))) {
            int64_t lo = tptr[col];
            for (int64_t i = 0; i < M; ++i) {
                int64_t hi = 0;
                if (lane == 0) hi = lower_bound_i32(tidx, lo, tptr[col + 1], row_bounds[i + 1]);
                hi = __shfl_sync(0xffffffffu, hi, 0);
                if (rsel.has(i)) {
                    double s = 0.0;
                    for (int64_t k = lo + lane; k < hi; k += 32) s = fma((double)tval[k], r[tidx[k]], s);
                    s = warp_sum(s);
                    acc = rn_add(acc, s);
                }
                lo = hi;
            }
        }
        if (lane == 0) g[col] = 2.0 * acc;
    }
}

}  // namespace bsgd
