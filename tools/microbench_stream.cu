// Does streaming the CSR arrays through the LSU cost gather throughput?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_stream tools/microbench_stream.cu && tools/mb_stream
//
// Every thread performs random 8-byte gathers from a 4 MB table (configs[1]'s
// x).  Variants add the matrix stream of the forward CSR kernel next to them:
//   * none        : gathers only (the ceiling measured in r01_gather_microbench.md)
//   * ldg         : 2 x 16-byte ld.global.nc.L1::no_allocate per 4 gathers (K1's vec4 path)
//   * tma         : the same bytes moved by cp.async.bulk into a shared-memory ring
//                   (one elected thread, mbarrier completion), read back with LDS.128
#include <cstdint>
#include <cstdio>

constexpr int THREADS = 256;
constexpr int ITERS = 4096;  // gathers per thread
constexpr int UNROLL = 8;

__device__ __forceinline__ uint32_t xs(uint32_t &s) {
    s ^= s << 13; s ^= s >> 17; s ^= s << 5;
    return s;
}

__device__ __forceinline__ int4 ld_nc4(const int4 *p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(THREADS) kern(const double *__restrict__ tab, uint32_t mask,
                                                const int4 *__restrict__ stream, double *out) {
    // MODE 0 none, 1 ldg stream
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * THREADS + threadIdx.x) * 2654435761u;
    double acc = 0.0;
    int sacc = 0;
    // each CTA streams its own contiguous region: ITERS/4*2 int4 per thread
    const int4 *sp = stream + (size_t)blockIdx.x * (ITERS / 2) * THREADS + threadIdx.x;
    for (int i = 0; i < ITERS; i += UNROLL) {
        double v[UNROLL];
        if (MODE == 1) {
            // UNROLL/4*2 = 4 stream loads per 8 gathers
#pragma unroll
            for (int u = 0; u < UNROLL / 2; ++u) {
                const int4 q = ld_nc4(sp);
                sp += THREADS;
                sacc += q.x ^ q.w;
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = __ldg(tab + ((xs(s) ^ (uint32_t)sacc) & mask));
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u];
    }
    out[blockIdx.x * THREADS + threadIdx.x] = acc + sacc;
}

// MODE 2: TMA ring.  Stage = THREADS * 4 int4 (16 KB), the bytes of 8 iterations' worth of stream.
constexpr int STAGE_INT4 = THREADS * (UNROLL / 2);
constexpr int NST = 4;

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(b)),
        "r"(ph));
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b))
                 : "memory");
}

__global__ void __launch_bounds__(THREADS) kern_tma(const double *__restrict__ tab, uint32_t mask,
                                                    const int4 *__restrict__ stream, double *out) {
    extern __shared__ int4 ring[];  // NST * STAGE_INT4
    __shared__ uint64_t bars[NST];
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * THREADS + threadIdx.x) * 2654435761u;
    const int4 *base = stream + (size_t)blockIdx.x * (ITERS / 2) * THREADS;
    const int steps = ITERS / UNROLL;
    if (threadIdx.x == 0) {
        for (int k = 0; k < NST; ++k) mbar_init(&bars[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < NST && k < steps; ++k) {
            mbar_expect(&bars[k], STAGE_INT4 * 16);
            bulk(ring + k * STAGE_INT4, base + (size_t)k * STAGE_INT4, STAGE_INT4 * 16, &bars[k]);
        }
    double acc = 0.0;
    int sacc = 0;
    for (int st = 0; st < steps; ++st) {
        const int slot = st % NST;
        mbar_wait(&bars[slot], (st / NST) & 1);
#pragma unroll
        for (int u = 0; u < UNROLL / 2; ++u) {
            const int4 q = ring[slot * STAGE_INT4 + u * THREADS + threadIdx.x];
            sacc += q.x ^ q.w;
        }
        double v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = __ldg(tab + ((xs(s) ^ (uint32_t)sacc) & mask));
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u];
        __syncthreads();  // slot free
        if (threadIdx.x == 0 && st + NST < steps) {
            mbar_expect(&bars[slot], STAGE_INT4 * 16);
            bulk(ring + slot * STAGE_INT4, base + (size_t)(st + NST) * STAGE_INT4, STAGE_INT4 * 16, &bars[slot]);
        }
    }
    out[blockIdx.x * THREADS + threadIdx.x] = acc + sacc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ghz = clk / 1e6;
    double *tab, *out;
    int4 *stream;
    const uint32_t mask = (1u << 19) - 1;  // 4 MB
    cudaMalloc(&tab, sizeof(double) << 19);
    cudaMemset(tab, 0, sizeof(double) << 19);
    for (int cpsm : {4, 8}) {
        const int grid = sms * cpsm;
        const size_t n4 = (size_t)grid * (ITERS / 2) * THREADS;
        cudaMalloc(&stream, n4 * 16);
        cudaMemset(stream, 0, n4 * 16);
        cudaMalloc(&out, sizeof(double) * grid * THREADS);
        cudaFuncSetAttribute(kern_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, NST * STAGE_INT4 * 16);
        for (int mode = 0; mode < 3; ++mode) {
            auto launch = [&]() {
                if (mode == 0) kern<0><<<grid, THREADS>>>(tab, mask, stream, out);
                else if (mode == 1) kern<1><<<grid, THREADS>>>(tab, mask, stream, out);
                else kern_tma<<<grid, THREADS, NST * STAGE_INT4 * 16>>>(tab, mask, stream, out);
            };
            launch();
            cudaDeviceSynchronize();
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int k = 0; k < 5; ++k) launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 5;
            cudaError_t e = cudaGetLastError();
            const double gathers = (double)grid * THREADS * ITERS;
            const double sbytes = mode ? (double)n4 * 16 : 0.0;
            printf("%d CTA/SM  %-5s %8.3f ms  %6.3f gathers/SM/cycle  stream %7.1f GB/s  %s\n", cpsm,
                   mode == 0 ? "none" : mode == 1 ? "ldg" : "tma", ms, gathers / (ms * 1e-3) / sms / (ghz * 1e9),
                   sbytes / (ms * 1e6), e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
        cudaFree(stream);
        cudaFree(out);
    }
    return 0;
}
