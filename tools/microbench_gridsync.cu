// Grid-wide exchange latency on B200: cooperative-groups grid.sync() around a partial-sum
// exchange (what csrc/fgp2.cu does once per FGP iteration) against a tagged exchange
// (each CTA publishes (value, tag) pairs with 16-byte stores after a fence; readers
// spin on the tags with acquire loads -- no counter, no second round trip).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_gridsync tools/microbench_gridsync.cu
//   tools/mb_gridsync [ctas=128] [threads=512] [rounds=2000]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int K = 5;

__global__ void k_gridsync(double *buf, double *out, int rounds) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double tot[K];
    double acc = 0.0;
    for (int r = 0; r < rounds; ++r) {
        double *b = buf + (size_t)(r & 1) * gridDim.x * K;
        __syncthreads();
        if (warp < K && lane == 0) b[blockIdx.x * K + warp] = (double)(r + blockIdx.x + warp);
        grid.sync();
        if (warp < K) {
            double v = 0.0;
            for (int c = lane; c < (int)gridDim.x; c += 32) v += b[c * K + warp];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) tot[warp] = v;
        }
        __syncthreads();
        acc += tot[0] + tot[K - 1];
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

struct alignas(16) Tagged {
    double v;
    unsigned long long tag;
};

__device__ __forceinline__ Tagged ld_acquire(const Tagged *p) {
    Tagged t;
    unsigned long long a, b;
    asm volatile("ld.acquire.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    t.v = __longlong_as_double((long long)a);
    t.tag = b;
    return t;
}
__device__ __forceinline__ Tagged ld_relaxed(const Tagged *p) {
    Tagged t;
    unsigned long long a, b;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    t.v = __longlong_as_double((long long)a);
    t.tag = b;
    return t;
}
__device__ __forceinline__ void st_release(Tagged *p, double v, unsigned long long tag) {
    asm volatile("st.release.gpu.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v)),
                 "l"(tag)
                 : "memory");
}

__global__ void k_tagged(Tagged *buf, double *out, int rounds, unsigned long long gen) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double tot[K];
    double acc = 0.0;
    for (int r = 0; r < rounds; ++r) {
        Tagged *b = buf + (size_t)(r & 1) * gridDim.x * K;
        const unsigned long long tag = gen * (1ull << 32) + (unsigned)r + 1;
        __syncthreads();   // the CTA's earlier global writes happen before the publishing lanes' release
        if (warp < K && lane == 0) st_release(&b[blockIdx.x * K + warp], (double)(r + blockIdx.x + warp), tag);
        if (warp < K) {
            // the lane's entries loaded together (independent relaxed loads), retried until
            // every tag is current, then one acquire fence
            double v = 0.0;
            const int n = ((int)gridDim.x - lane + 31) / 32;
            Tagged t[8];
            bool ok;
            do {
                ok = true;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < n) t[q] = ld_relaxed(&b[(lane + 32 * q) * K + warp]);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < n) ok &= t[q].tag == tag;
            } while (!ok);
            __threadfence();
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < n) v += t[q].v;
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) tot[warp] = v;
        }
        __syncthreads();
        acc += tot[0] + tot[K - 1];
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main(int argc, char **argv) {
    int ctas = argc > 1 ? atoi(argv[1]) : 128, threads = argc > 2 ? atoi(argv[2]) : 512;
    int rounds = argc > 3 ? atoi(argv[3]) : 2000;
    double *buf, *out;
    Tagged *tb;
    cudaMalloc(&buf, sizeof(double) * 2 * ctas * K);
    cudaMalloc(&tb, sizeof(Tagged) * 2 * ctas * K);
    cudaMemset(tb, 0, sizeof(Tagged) * 2 * ctas * K);
    cudaMalloc(&out, sizeof(double) * ctas);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    double h1[1024], h2[1024];
    for (int rep = 0; rep < 3; ++rep) {
        void *args[] = {&buf, &out, &rounds};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)k_gridsync, dim3(ctas), dim3(threads), args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h1, out, sizeof(double) * ctas, cudaMemcpyDeviceToHost);
        printf("grid.sync exchange : %.3f us per round (%s)\n", ms * 1e3 / rounds, cudaGetErrorString(cudaGetLastError()));
        unsigned long long gen = rep + 1;
        void *targs[] = {&tb, &out, &rounds, &gen};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)k_tagged, dim3(ctas), dim3(threads), targs, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h2, out, sizeof(double) * ctas, cudaMemcpyDeviceToHost);
        printf("tagged exchange    : %.3f us per round (%s) %s\n", ms * 1e3 / rounds, cudaGetErrorString(cudaGetLastError()),
               h1[0] == h2[0] && h1[ctas - 1] == h2[ctas - 1] ? "same sums" : "MISMATCH");
    }
    return 0;
}
