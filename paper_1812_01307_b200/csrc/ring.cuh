// TMA-staged form of the blocked CSR product (spmv.cuh csr_blocked_kernel, 16 lanes
// per row, compressed indices).
//
// csr_blocked_kernel holds every in-flight stream load in registers: two blocks per
// lane, 48 warps per SM, and ncu shows all stalls on the long scoreboard with DRAM at
// two thirds of its peak (profiles/r02_k1_k2_blocked.md) -- the kernel is bound by the
// bytes it can keep in flight, not by L1 or HBM.  Here the stream is stored as one
// contiguous record per 64-entry block
//
//     [ int2 half bases | 8 B pad | uint16 off[64] | V val[64] ]     (400 B for float32)
//
// in row order, and each half-warp (16 lanes = one row at a time) owns a ring of S
// records in shared memory that its first lane keeps full with 1-D TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), running ahead across row boundaries.  The
// consumer lanes read their 8 bytes of offsets and 16 bytes of values from the ring,
// gather from the (tile-ordered) vector and sum exactly as csr_blocked_kernel does:
// lane l takes the entries = l mod 16 in order, same shuffle tree -- bit-identical.
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace bsgd {

constexpr int kRingLanes = 16;                // lanes per row
constexpr int kRingBlock = 4 * kRingLanes;    // entries per record

template <typename V>
__host__ __device__ constexpr int ring_rec_bytes() {
    return 16 + 2 * kRingBlock + (int)sizeof(V) * kRingBlock;
}

template <typename V>
struct CsrR {
    int64_t nrows;
    const int64_t *bptr;          // [nrows + 1] first record of each row
    const unsigned char *rec;     // records, ring_rec_bytes<V>() each
    const double *vec;
};

// pack the blocked arrays (spmv.cuh CsrB with 16 lanes, compressed) into records:
// one thread per 16-byte unit
template <typename V>
__global__ void ring_pack_kernel(int64_t nblocks, const int2 *half, const uint16_t *off, const V *val,
                                 unsigned char *rec) {
    constexpr int REC = ring_rec_bytes<V>(), UNITS = REC / 16, OFFU = 2 * kRingBlock / 16;
    const int64_t total = nblocks * UNITS;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = u / UNITS;
        const int k = (int)(u - b * UNITS);
        int4 v;
        if (k == 0) {
            const int2 h = half[b];
            v = make_int4(h.x, h.y, 0, 0);
        } else if (k <= OFFU) {
            v = reinterpret_cast<const int4 *>(off + b * kRingBlock)[k - 1];
        } else {
            v = reinterpret_cast<const int4 *>(val + b * kRingBlock)[k - 1 - OFFU];
        }
        reinterpret_cast<int4 *>(rec + b * REC)[k] = v;
    }
}

__global__ void ring_bptr_kernel(int64_t n, const int64_t *ptr, int64_t *bptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bptr[i] = ptr[i] / kRingBlock;
}

template <typename V>
__device__ __forceinline__ void ring_vals(const unsigned char *r, int hl, double (&v)[4]) {
    if constexpr (sizeof(V) == 4) {
        const float4 a = *reinterpret_cast<const float4 *>(r + 16 + 2 * kRingBlock + 16 * hl);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
        const double2 a = *reinterpret_cast<const double2 *>(r + 16 + 2 * kRingBlock + 32 * hl);
        const double2 b = *reinterpret_cast<const double2 *>(r + 16 + 2 * kRingBlock + 32 * hl + 16);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
}

__device__ __forceinline__ int4 ring_cols(const unsigned char *r, int hl) {
    const int2 h = *reinterpret_cast<const int2 *>(r);
    const uint2 d = *reinterpret_cast<const uint2 *>(r + 16 + 8 * hl);
    return make_int4(h.x + (int32_t)(d.x & 0xFFFFu), h.x + (int32_t)(d.x >> 16), h.y + (int32_t)(d.y & 0xFFFFu),
                     h.y + (int32_t)(d.y >> 16));
}

template <typename V, int S>
constexpr size_t ring_smem_bytes() {
    return (size_t)(kThreads / kRingLanes) * S * ring_rec_bytes<V>();
}

template <typename V, int S, class Epi>
__global__ void __launch_bounds__(kThreads) csr_ring_kernel(CsrR<V> A, Epi epi, double *part, int64_t *cnt) {
    static_assert((S & (S - 1)) == 0, "ring depth must be a power of two");
    constexpr int REC = ring_rec_bytes<V>();
    constexpr int HW = kThreads / kRingLanes;   // half-warps (rows in flight) per CTA
    extern __shared__ __align__(128) unsigned char ring_smem[];
    __shared__ uint64_t bars[HW * S];
    __shared__ double sm[8 * (kThreads / 32)];
    const int lane = threadIdx.x & 31, hl = lane & 15, hw = threadIdx.x >> 4;
    const unsigned hmask = 0xFFFFu << (lane & 16);
    unsigned char *ring = ring_smem + (size_t)hw * S * REC;
    uint64_t *bar = bars + hw * S;
    if (hl == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const double *__restrict__ vec = A.vec;
    // row of this half-warp: the two halves of a warp take adjacent rows (csr_blocked_kernel's map)
    const int64_t stride = (int64_t)gridDim.x * HW;
    const int64_t first = (int64_t)blockIdx.x * HW + hw;
    // producer: the half-warp's records in consumption order, S ahead of the consumer
    int64_t prow = first, pb = 0, pe = 0;
    if (prow < A.nrows) {
        pb = A.bptr[prow];
        pe = A.bptr[prow + 1];
    }
    uint32_t pq = 0;
    auto produce = [&]() {
        while (prow < A.nrows && pb == pe) {
            prow += stride;
            if (prow < A.nrows) {
                pb = A.bptr[prow];
                pe = A.bptr[prow + 1];
            }
        }
        if (prow < A.nrows) {
            if (hl == 0) {
                const uint32_t st = pq & (S - 1);
                mbar_arrive_expect_tx(&bar[st], REC);
                bulk_g2s(ring + st * REC, A.rec + pb * REC, REC, &bar[st]);
            }
            ++pb;
            ++pq;
        }
    };
#pragma unroll
    for (int i = 0; i < S; ++i) produce();
    uint32_t cq = 0;
    for (int64_t row = first; row < A.nrows; row += stride) {
        const int64_t nb = A.bptr[row + 1] - A.bptr[row];
        double s = 0.0;
        for (int64_t b = 0; b < nb; b += 2) {
            const bool two = b + 1 < nb;
            const unsigned char *r0 = ring + (cq & (S - 1)) * REC;
            const unsigned char *r1 = ring + ((cq + 1) & (S - 1)) * REC;
            mbar_wait(&bar[cq & (S - 1)], (cq / S) & 1);
            const int4 ca = ring_cols(r0, hl);
            double va[4];
            ring_vals<V>(r0, hl, va);
            const double xa0 = __ldg(vec + ca.x), xa1 = __ldg(vec + ca.y), xa2 = __ldg(vec + ca.z),
                         xa3 = __ldg(vec + ca.w);
            if (two) {
                mbar_wait(&bar[(cq + 1) & (S - 1)], ((cq + 1) / S) & 1);
                const int4 cb = ring_cols(r1, hl);
                double vb[4];
                ring_vals<V>(r1, hl, vb);
                const double xb0 = __ldg(vec + cb.x), xb1 = __ldg(vec + cb.y), xb2 = __ldg(vec + cb.z),
                             xb3 = __ldg(vec + cb.w);
                s = fma(va[0], xa0, s); s = fma(va[1], xa1, s); s = fma(va[2], xa2, s); s = fma(va[3], xa3, s);
                s = fma(vb[0], xb0, s); s = fma(vb[1], xb1, s); s = fma(vb[2], xb2, s); s = fma(vb[3], xb3, s);
            } else {
                s = fma(va[0], xa0, s); s = fma(va[1], xa1, s); s = fma(va[2], xa2, s); s = fma(va[3], xa3, s);
            }
            __syncwarp(hmask);   // every lane has consumed the records: their slots may be refilled
            produce();
            if (two) produce();
            cq += two ? 2 : 1;
        }
#pragma unroll
        for (int off = kRingLanes / 2; off > 0; off >>= 1) s += __shfl_xor_sync(hmask, s, off, kRingLanes);
        if (hl == 0) epi(row, s);
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

}  // namespace bsgd
