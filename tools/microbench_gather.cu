// Random-gather throughput on B200: global (L2-resident table) vs local shared
// memory vs distributed shared memory across a thread-block cluster.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_gather.cu && ./mb
//
// Each thread performs ITERS dependent-free random 8-byte loads (xorshift
// indices), sums them, and writes one value.  Reported: loads per second and
// per SM per cycle (at the observed SM clock).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

constexpr int THREADS = 256;
constexpr int ITERS = 4096;
constexpr int UNROLL = 8;

__device__ __forceinline__ uint32_t xs(uint32_t &s) {
    s ^= s << 13; s ^= s >> 17; s ^= s << 5;
    return s;
}

__global__ void gather_global(const double *__restrict__ tab, uint32_t mask, double *out) {
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * THREADS + threadIdx.x) * 2654435761u;
    double acc = 0.0;
    for (int i = 0; i < ITERS; i += UNROLL) {
        double v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = __ldg(tab + (xs(s) & mask));
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u];
    }
    out[blockIdx.x * THREADS + threadIdx.x] = acc;
}

template <int WORDS>
__global__ void gather_smem(double *out) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < WORDS; i += THREADS) sm[i] = i * 0.5;
    __syncthreads();
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * THREADS + threadIdx.x) * 2654435761u;
    double acc = 0.0;
    for (int i = 0; i < ITERS; i += UNROLL) {
        double v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = sm[xs(s) & (WORDS - 1)];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u];
    }
    out[blockIdx.x * THREADS + threadIdx.x] = acc;
}

template <int WORDS, int CL>
__global__ void gather_dsmem(double *out) {
    extern __shared__ double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    for (int i = threadIdx.x; i < WORDS; i += THREADS) sm[i] = i * 0.5;
    cluster.sync();
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * THREADS + threadIdx.x) * 2654435761u;
    double acc = 0.0;
    double *peers[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) peers[r] = cluster.map_shared_rank(sm, r);
    for (int i = 0; i < ITERS; i += UNROLL) {
        double v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const uint32_t h = xs(s);
            v[u] = peers[(h >> 24) % CL][h & (WORDS - 1)];
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u];
    }
    cluster.sync();
    out[blockIdx.x * THREADS + threadIdx.x] = acc;
}

static float timeit(void (*launch)(void *), void *arg) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(arg);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return ms / 5;
}

struct Ctx { double *tab; double *out; uint32_t mask; int grid; };
static Ctx C;

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ghz = clk / 1e6;
    cudaMalloc(&C.tab, sizeof(double) * (1 << 22));
    cudaMemset(C.tab, 0, sizeof(double) * (1 << 22));
    cudaMalloc(&C.out, sizeof(double) * 148 * 64 * THREADS);
    auto report = [&](const char *name, float ms, long long blocks) {
        const double loads = (double)blocks * THREADS * ITERS;
        printf("%-40s %8.3f ms  %8.1f Gload/s  %6.2f load/SM/cycle (at %.2f GHz max)\n", name, ms,
               loads / ms / 1e6, loads / (ms * 1e-3) / sms / (ghz * 1e9), ghz);
    };
    for (int words_log : {16, 19, 22}) {  // 512 KB, 4 MB, 32 MB tables
        C.mask = (1u << words_log) - 1;
        C.grid = sms * 8;
        float ms = timeit([](void *) { gather_global<<<C.grid, THREADS>>>(C.tab, C.mask, C.out); }, nullptr);
        char nm[64];
        snprintf(nm, 64, "global table %d KB", (int)((8ll << words_log) >> 10));
        report(nm, ms, C.grid);
    }
    {
        constexpr int W = 16384;  // 128 KB
        cudaFuncSetAttribute(gather_smem<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 8);
        C.grid = sms;
        float ms = timeit([](void *) { gather_smem<W><<<C.grid, THREADS, W * 8>>>(C.out); }, nullptr);
        report("local smem 128 KB, 1 CTA/SM", ms, C.grid);
        C.grid = sms * 1;
    }
    {
        constexpr int W = 4096;  // 32 KB, 4 CTA/SM
        C.grid = sms * 4;
        float ms = timeit([](void *) { gather_smem<W><<<C.grid, THREADS, W * 8>>>(C.out); }, nullptr);
        report("local smem 32 KB, 4 CTA/SM", ms, C.grid);
    }
    {
        constexpr int W = 16384;
        constexpr int CL = 8;
        cudaFuncSetAttribute(gather_dsmem<W, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 8);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(144);
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = W * 8;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        static cudaLaunchConfig_t S; S = cfg;
        float ms = timeit([](void *) { cudaLaunchKernelEx(&S, gather_dsmem<16384, 8>, C.out); }, nullptr);
        report("DSMEM cluster 8 x 128 KB", ms, 144);
    }
    {
        constexpr int W = 16384;
        constexpr int CL = 16;
        cudaFuncSetAttribute(gather_dsmem<W, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 8);
        cudaFuncSetAttribute(gather_dsmem<W, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(144);
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = W * 8;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        static cudaLaunchConfig_t S; S = cfg;
        float ms = timeit([](void *) { cudaLaunchKernelEx(&S, gather_dsmem<16384, 16>, C.out); }, nullptr);
        report("DSMEM cluster 16 x 128 KB", ms, 144);
    }
    return 0;
}
