// Can the TMA unit gather the SpMV's random vector elements faster than the
// LSU?  LDG gathers are capped near one distinct sector per SM per cycle by the
// L1 tag stage (profiles/r01_gather_microbench.md).  TMA requests bypass the
// L1TEX pipeline, so this measures, on a 4 MB table (configs[1]'s x):
//
//   * tile::gather4 (2-D tensor map, 4 arbitrary rows per instruction) with
//     16-byte and 32-byte rows, 1..8 issuing warps per CTA;
//   * 1-D cp.async.bulk of one 16-byte pair per element;
//   * LDG baselines (.nc, .cg) and random red.global.add.f64 (the scatter a
//     single-pass forward+transposed kernel would need).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tmagather \
//        tools/microbench_tma_gather.cu -lcuda && ./tools/mb_tmagather
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "../paper_1812_01307_b200/csrc/sm100.cuh"

using namespace bsgd;

constexpr int ROWS_LOG = 19;  // 512 K elements of 8 B = 4 MB
constexpr int STEPS = 512;    // slots consumed per warp
constexpr int G = 8;          // gather4 ops per slot -> 32 rows, one per lane
constexpr int DEPTH = 8;      // slots in flight per warp

__device__ __forceinline__ uint32_t xs(uint32_t &s) {
    s ^= s << 13; s ^= s >> 17; s ^= s << 5;
    return s;
}

__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *map, int c0, int r0, int r1, int r2, int r3,
                                        uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// W doubles per tensor row; each warp runs its own DEPTH-slot ring.
template <int W, int MODE>  // MODE 0: gather4, 1: 1-D bulk copy of W doubles per element
__global__ void tma_gather(const __grid_constant__ CUtensorMap map, const double *tab, double *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // gather4 destinations must be 128-byte aligned: one 128 B cell per op
    constexpr int OPB = (MODE == 0 && 4 * W * 8 < 128) ? 128 : 4 * W * 8;
    constexpr int SLOT_BYTES = G * OPB;
    unsigned char *ring = sm + 1024 + warp * DEPTH * SLOT_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm) + warp * DEPTH;
    if (lane == 0)
        for (int d = 0; d < DEPTH; ++d) mbar_init(full + d, 1);
    fence_mbar_init();
    __syncwarp();
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    const uint32_t mask = (1u << ROWS_LOG) / W - 1;
    auto issue = [&](int slot) {
        // every lane draws its own row; lane 0 issues all the copies
        const uint32_t row = xs(s) & mask;
        if (lane == 0) mbar_arrive_expect_tx(full + slot, G * 4 * W * 8);
        __syncwarp();
        unsigned char *dst = ring + slot * SLOT_BYTES;
        if (MODE == 0) {
#pragma unroll
            for (int k = 0; k < G; ++k) {
                const int r0 = __shfl_sync(~0u, row, 4 * k), r1 = __shfl_sync(~0u, row, 4 * k + 1);
                const int r2 = __shfl_sync(~0u, row, 4 * k + 2), r3 = __shfl_sync(~0u, row, 4 * k + 3);
                if (lane == 0) gather4(dst + k * OPB, &map, 0, r0, r1, r2, r3, full + slot);
            }
        } else {
            // each lane issues its own 1-D bulk copy (32 issuing lanes)
            bulk_g2s(dst + lane * W * 8, tab + (size_t)row * W, W * 8, full + slot);
        }
    };
    for (int d = 0; d < DEPTH; ++d) issue(d);
    double acc = 0.0;
    for (int st = 0; st < STEPS; ++st) {
        const int slot = st % DEPTH;
        mbar_wait(full + slot, (st / DEPTH) & 1);
        acc += reinterpret_cast<const double *>(ring + slot * SLOT_BYTES + (lane >> 2) * OPB)[(lane & 3) * W];
        __syncwarp();
        if (st + DEPTH < STEPS) issue(slot);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>  // 0: ld.global.nc, 1: ld.global.cg, 2: red.global.add.f64
__global__ void lsu_kernel(double *tab, double *out) {
    uint32_t s = 0x9E3779B9u ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    const uint32_t mask = (1u << ROWS_LOG) - 1;
    double acc = 0.0;
    for (int i = 0; i < 4096; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double *p = tab + (xs(s) & mask);
            if (MODE == 0) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v[u]) : "l"(p));
            else if (MODE == 1) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v[u]) : "l"(p));
            else { asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(1.0) : "memory"); v[u] = 0; }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncodeFn enc, double *tab, int w) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)((1u << ROWS_LOG) / w)};
    cuuint64_t strides[1] = {(cuuint64_t)w * 8};
    cuuint32_t box[2] = {(cuuint32_t)w, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, tab, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d (w=%d)\n", (int)r, w);
    return m;
}

int main(int argc, char **argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;  // run one variant (a fault is sticky)
    int id = 0;
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double hz = clk * 1e3;
    double *tab, *out;
    cudaMalloc(&tab, 8ull << ROWS_LOG);
    cudaMemset(tab, 0, 8ull << ROWS_LOG);
    cudaMalloc(&out, 8ull * sms * 4096);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timed = [&](const char *name, double items, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int k = 0; k < 5; ++k) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        cudaError_t e = cudaGetLastError();
        printf("%-46s %8.3f ms  %7.3f elem/SM/cycle  %s\n", name, ms, items / (ms * 1e-3) / sms / hz,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    auto run_tma = [&](auto kern, int w, int mode, int warps, int ctas_per_sm) {
        if (only >= 0 && id++ != only) return;
        CUtensorMap m = make_map(enc, tab, w);
        const int smem = 1024 + warps * DEPTH * G * (mode == 0 && 4 * w * 8 < 128 ? 128 : 4 * w * 8);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = sms * ctas_per_sm;
        char nm[96];
        snprintf(nm, 96, "%s W=%d B, %d warps x %d CTA/SM", mode == 0 ? "gather4" : "bulk 1-D", w * 8, warps,
                 ctas_per_sm);
        timed(nm, (double)grid * warps * STEPS * 32, [&] { kern<<<grid, warps * 32, smem>>>(m, tab, out); });
    };
    for (int warps : {1, 4, 8})
        for (int cps : {1, 2}) {
            run_tma(tma_gather<2, 0>, 2, 0, warps, cps);
            run_tma(tma_gather<4, 0>, 4, 0, warps, cps);
            run_tma(tma_gather<2, 1>, 2, 1, warps, cps);
        }
    const int grid = sms * 8;
    if (only >= 0 && only < 18) return 0;
    timed("LDG.nc random 8 B", (double)grid * 256 * 4096, [&] { lsu_kernel<0><<<grid, 256>>>(tab, out); });
    timed("LDG.cg random 8 B", (double)grid * 256 * 4096, [&] { lsu_kernel<1><<<grid, 256>>>(tab, out); });
    timed("RED.add.f64 random 8 B", (double)grid * 256 * 4096, [&] { lsu_kernel<2><<<grid, 256>>>(tab, out); });
    return 0;
}
