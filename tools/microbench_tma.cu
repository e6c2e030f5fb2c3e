// Latency / throughput of the panel pipeline used by the tiled SpMV, isolated:
// every CTA walks `steps` panels through a 2..NSLOT-slot buffer; a panel is
// either TMA-bulk-copied by each CTA itself or multicast by the cluster
// leader after all members released the slot.  Consumers do no work, so the
// time per step is the pipeline's own cost.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_tma tools/microbench_tma.cu
#include <cstdio>
#include <cstdint>

#include "../paper_1812_01307_b200/csrc/sm100.cuh"

using namespace bsgd;

template <int CL, bool MC, int NSLOT>
__global__ void __launch_bounds__(64, 1) panel_pipe(const double *vec, int64_t ncols, int P, int steps, double *out) {
    extern __shared__ __align__(128) unsigned char smem[];
    double *buf = reinterpret_cast<double *>(smem);
    uint64_t *bars = reinterpret_cast<uint64_t *>(buf + (size_t)NSLOT * P);
    uint64_t *full = bars, *freeb = bars + NSLOT, *clus = bars + 2 * NSLOT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSLOT; ++s) { mbar_init(full + s, 1); mbar_init(freeb + s, 1); mbar_init(clus + s, CL); }
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();
    const int NP = (int)(ncols / P);
    double acc = 0.0;
    if (warp == 0) {
        if (lane == 0) {
            for (int q = 0; q < steps; ++q) {
                const int s = q % NSLOT;
                const uint32_t bytes = (uint32_t)P * 8;
                const double *src = vec + (size_t)(q % NP) * P;
                if (q >= NSLOT) mbar_wait(freeb + s, ((q / NSLOT) - 1) & 1);
                mbar_arrive_expect_tx(full + s, bytes);
                if (MC) {
                    mbar_arrive_remote(clus + s, 0);
                    if (rank == 0) {
                        mbar_wait_cluster(clus + s, (q / NSLOT) & 1);
                        bulk_g2s_multicast(buf + (size_t)s * P, src, bytes, full + s, (uint16_t)((1u << CL) - 1));
                    }
                } else {
                    bulk_g2s(buf + (size_t)s * P, src, bytes, full + s);
                }
            }
        }
        __syncwarp();
    } else {
        for (int q = 0; q < steps; ++q) {
            const int s = q % NSLOT;
            mbar_wait(full + s, (q / NSLOT) & 1);
            acc += buf[(size_t)s * P + lane];
            __syncwarp();
            if (lane == 0) mbar_arrive(freeb + s);
        }
    }
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x == 32) out[blockIdx.x] = acc;
}

template <int CL, bool MC, int NSLOT>
static void run(const char *name, const double *vec, int64_t ncols, int P, int steps, double *out, int grid) {
    auto k = panel_pipe<CL, MC, NSLOT>;
    const size_t smem = (size_t)NSLOT * P * 8 + 3 * NSLOT * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, vec, ncols, P, steps, out);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k, vec, ncols, P, steps, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    const double per = ms * 1e3 / steps;
    const double gbs = (double)P * 8 * steps * (MC ? grid / CL : grid) / (ms * 1e-3) / 1e9;
    printf("%-44s P=%5d  %7.3f ms  %6.3f us/step  L2->SM %7.1f GB/s  %s\n", name, P, ms, per, gbs,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    const int64_t ncols = 1 << 19;
    double *vec, *out;
    cudaMalloc(&vec, ncols * 8);
    cudaMemset(vec, 0, ncols * 8);
    cudaMalloc(&out, 4096 * 8);
    const int steps = 2000;
    const int grid = 120;
    for (int P : {8192, 2048, 512}) {
        run<8, true, 2>("multicast cluster 8, 2 slots", vec, ncols, P, steps, out, grid);
        run<8, false, 2>("per-CTA bulk copy (cluster 8 launch), 2 slots", vec, ncols, P, steps, out, grid);
        run<1, false, 2>("per-CTA bulk copy, no cluster, 2 slots", vec, ncols, P, steps, out, grid);
    }
    run<8, true, 4>("multicast cluster 8, 4 slots", vec, ncols, 4096, steps, out, grid);
    run<8, true, 8>("multicast cluster 8, 8 slots", vec, ncols, 2048, steps, out, grid);
    run<1, false, 8>("per-CTA bulk copy, no cluster, 8 slots", vec, ncols, 2048, steps, out, grid);
    run<2, true, 4>("multicast cluster 2, 4 slots", vec, ncols, 4096, steps, out, grid);
    run<4, true, 4>("multicast cluster 4, 4 slots", vec, ncols, 4096, steps, out, grid);
    return 0;
}
