// Time the 3-D FGP phases separately at 256^3 (tools/microbench_prox_phases.cu):
//   A   candidate c = proj(q + step grad(b + w div q))     (fgp.cuh candidate())
//   BC  dual value + momentum commit terms                  (DualCommitTerms, as a plain sweep)
//   copy 7-field streaming reference (read 4 fields, write 3) = phase A's HBM traffic
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1812_01307_b200/csrc \
//        -o tools/mb_prox tools/microbench_prox_phases.cu && tools/mb_prox
#include <cstdio>
#include <vector>

#include "fgp.cuh"

using namespace bsgd;

__global__ void __launch_bounds__(kThreads, 2) phase_a(ProxArgs a) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
    double *Q[3] = {a.f[3], a.f[4], a.f[5]}, *C[3] = {a.f[6], a.f[7], a.f[8]};
    for (int64_t p0 = tid; p0 < a.N; p0 += 2 * nthr) {
        const int64_t p1 = p0 + nthr;
        double c0[3], c1[3];
        candidate<3>(a, Q, p0, c0);
        if (p1 < a.N) candidate<3>(a, Q, p1, c1);
        for (int k = 0; k < 3; ++k) C[k][p0] = c0[k];
        if (p1 < a.N)
            for (int k = 0; k < 3; ++k) C[k][p1] = c1[k];
    }
}

__global__ void __launch_bounds__(kThreads, 2) phase_bc(ProxArgs a, double *sink) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
    DualCommitTerms<3> f;
    f.b = a.b; f.w = a.w; f.D = a.D; f.H = a.H; f.W = a.W; f.beta = 0.3;
    for (int k = 0; k < 3; ++k) { f.C[k] = a.f[6 + k]; f.P[k] = a.f[k]; f.Q[k] = a.f[3 + k]; }
    double acc = 0.0;
    for (int64_t p = tid; p < a.N; p += nthr) {
        double t[7];
        f(p, t);
        acc += t[0] + t[1] + t[4];
    }
    if (acc == 12345.0) sink[0] = acc;
}

__global__ void __launch_bounds__(kThreads, 2) copy7(ProxArgs a) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = tid; p < a.N; p += nthr) {
        const double s = a.b[p] + a.f[3][p] + a.f[4][p] + a.f[5][p];
        a.f[6][p] = s; a.f[7][p] = s * 2; a.f[8][p] = s * 3;
    }
}

int main() {
    const int64_t D = 256, H = 256, W = 256, N = D * H * W;
    double *buf;
    cudaMalloc(&buf, sizeof(double) * N * 10);
    cudaMemset(buf, 0, sizeof(double) * N * 10);
    double *sink;
    cudaMalloc(&sink, 8);
    ProxArgs a = {};
    a.D = D; a.H = H; a.W = W; a.N = N;
    a.b = buf + 9 * N;
    for (int k = 0; k < 9; ++k) a.f[k] = buf + k * N;
    a.w = 0.05; a.step = 1.0 / (12 * 0.05);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto timeit = [&](auto launch, const char *name, double bytes) {
        launch();
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        printf("%-6s %8.3f ms  %7.1f GB/s (algorithmic)  %s\n", name, ms, bytes / (ms * 1e6),
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int grid : {256, 296, 592, 1184}) {
        printf("grid %d\n", grid);
        timeit([&] { phase_a<<<grid, kThreads>>>(a); }, "A", 8.0 * N * 7);
        timeit([&] { phase_bc<<<grid, kThreads>>>(a, sink); }, "BC", 8.0 * N * 10);
        timeit([&] { copy7<<<grid, kThreads>>>(a); }, "copy7", 8.0 * N * 7);
    }
    return 0;
}
