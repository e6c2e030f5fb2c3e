// Slice-stacked operator for 3-D parallel-beam CT (configs[4], SURVEY.md §8 row f).
//
// configs[4]'s A is block-diagonal per slice with the same 2-D Siddon matrix
// A2 on every slice.  Stored as such it is ~1e10 nonzeros (~80 GB, twice that
// with A^T); stored as A2 (~4e7 nonzeros, ~0.3 GB) it fits next to everything
// else in one GPU's HBM.  The plan keeps A2 and A2^T and applies them to all
// slices at once in the INTERLEAVED order
//
//     row R = r * D + z,   column C = c * D + z,   A[R, C] = A2[r, c],
//
// i.e. A = A2 (x) I_D.  A product is then a sparse-times-tall-skinny product:
// one (c, A2[r, c]) entry is read once and applied to D contiguous vector
// values x[c*D .. c*D + D), so vector traffic is coalesced 8-byte-per-lane
// rows instead of random 8-byte gathers, and matrix traffic is D times
// smaller.  The solver vector's interleaved order maps to the z-major volume
// through the ordinary layout permutation (tv.VolumeLayout).
//
// Arithmetic order.  Every output is accumulated in the reference's exact
// order (oracle/bsgd_oracle.c, scipy's csr_matvec / csc_matvec restated):
// sequential products inside each block segment, one multiply and one add per
// term (no FMA), block segments folded in ascending block order -- so the
// stacked products, block products and pair products are bit-identical to the
// oracle's, and the K1 residual is y - z_0 - z_1 - ... exactly as
// assemble_residual (blockops.py:264-278).
//
// Work decomposition.  A work item is one stored row and a chunk of ZC = L*KZ
// slices: L lanes per row (L = min(32, pow2ceil(D))), KZ slices per lane,
// lane g handling z = z0 + g + L*s.  Items run chunk-major, so the warps in
// flight all read the same slice chunk of the vector and its working set
// (stored columns x ZC x 8 bytes) stays L2-resident; the host picks KZ to
// bound it.  The L lanes of a row read its entries with 16-byte broadcast
// loads (4 entries per request) and issue 4*KZ independent vector loads before
// the in-order multiply/add chain, so the loop is a few instructions per
// (entry, slice) rather than per-lane shuffles and index arithmetic.
#pragma once

#include "common.cuh"

namespace bsgd {

template <typename V>
struct Stk {
    int64_t nrows;           // stored rows (A2 rows for K1, A2^T rows for K2)
    const int64_t *ptr;
    const int32_t *idx;
    const V *val;
    const double *vec;       // interleaved input, indexed by the entry's interleaved index
    int64_t D;               // slices
    const int64_t *bounds;   // block bounds over the entries' interleaved index (col bounds for K1, row bounds for K2)
    const int64_t *sbounds;  // ALIGNED: the same bounds / D (every bound a multiple of D)
    int64_t nb;              // number of blocks
    const double *y;         // residual mode: measurements (interleaved rows)
    int L;                   // lanes per stored row (power of two <= 32)
};

// residual-mode epilogue target: the kernel already formed y - z_0 - z_1 - ...
struct EpiResidFinal {
    double *r;
    double acc = 0.0;
    static constexpr int K = 1;
    __device__ __forceinline__ void operator()(int64_t row, double v) {
        r[row] = v;
        acc += v * v;
    }
    __device__ __forceinline__ void flush(double *v) { v[0] = acc; }
};

// four consecutive entries (k 4-aligned) with 16-byte streaming loads; every
// lane of a row group reads the same addresses (one broadcast request)
template <typename V>
__device__ __forceinline__ void stk_load4(const int32_t *idx, const V *val, int64_t k, uint64_t pol, int32_t (&c)[4],
                                          double (&v)[4]) {
    const int4 c4 = ld_stream4(idx + k, pol);
    c[0] = c4.x; c[1] = c4.y; c[2] = c4.z; c[3] = c4.w;
    if constexpr (sizeof(V) == 4) {
        const float4 v4 = ld_stream4(reinterpret_cast<const float *>(val) + k, pol);
        v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
    } else {
        const double2 a = ld_stream2(reinterpret_cast<const double *>(val) + k, pol);
        const double2 b = ld_stream2(reinterpret_cast<const double *>(val) + k + 2, pol);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
}

// RESID = false: out = ((s_0 + s_1) + s_2) + ...   (blockops.py:237-243 / 254-260)
// RESID = true : out = ((y - s_0) - s_1) - ...     (assemble_residual)
// ALIGNED: every block bound is a multiple of D, so an entry's block depends on
//          its stored index only: one test per entry serves all slices.
//          Otherwise each slice keeps its own stored-index threshold
//          ceil((bound - z) / D), still one 32-bit compare per slice.
// W: one row per warp (L = 32) and D a multiple of 32*KZ: slice offsets are
//    compile-time and no slice predicates are needed.
// Interleaved indices are < 2^31 (checked at plan creation), so all index
// arithmetic is 32-bit.  Occupancy: 4 CTAs/SM (64 registers) wherever that
// costs no more than a few spills -- the loop is latency-bound on L2, so warps
// matter more than registers (configs[4] epoch 17.3 -> 14.2 ms); the unaligned
// plain product keeps 3 (it spills at 64).
template <typename V, int KZ, bool RESID, bool ALIGNED, bool W, class Epi>
__global__ void __launch_bounds__(kThreads, (ALIGNED || Epi::K == 4) ? 4 : 3) stacked_kernel(Stk<V> A, Epi epi, double *part, int64_t *cnt) {
    __shared__ double sm[8 * (kThreads / 32)];
    const int lane = threadIdx.x & 31;
    const int L = W ? 32 : A.L;
    const int rpw = 32 / L;
    const int sub = lane / L, gl = lane - sub * L;
    const int32_t D = (int32_t)A.D;
    const uint32_t D8 = 8u * (uint32_t)D;
    const int32_t ZC = L * KZ;
    const int64_t nchunks = (D + ZC - 1) / ZC;
    const int64_t ngroups = (A.nrows + rpw - 1) / rpw;
    const int64_t items = ngroups * nchunks;
    const int64_t nwarps = (int64_t)gridDim.x * (kThreads / 32);
    const uint64_t pol = policy_evict_first();
    const int32_t *__restrict__ idx = A.idx;
    const V *__restrict__ val = A.val;

    for (int64_t it = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); it < items; it += nwarps) {
        const int64_t ch = it / ngroups, grp = it - ch * ngroups;
        const int64_t r = grp * rpw + sub;
        const bool live = r < A.nrows;
        const int32_t zb = (int32_t)ch * ZC + gl;
        const double *__restrict__ xb = A.vec + zb;
        double seg[KZ], acc[KZ];
        int32_t thr[KZ];
        int jb[KZ];
        bool zok[KZ];
#pragma unroll
        for (int s = 0; s < KZ; ++s) {
            const int32_t z = zb + s * L;
            zok[s] = W ? live : (live && z < D);
            seg[s] = 0.0;
            acc[s] = (RESID && zok[s]) ? A.y[r * D + z] : 0.0;
            jb[s] = 0;
            if constexpr (ALIGNED) thr[s] = (int32_t)__ldg(A.sbounds + 1);
            else thr[s] = (int32_t)((__ldg(A.bounds + 1) - z + D - 1) / D);
        }
        auto fold = [&](int s) {
            if constexpr (RESID) acc[s] = rn_sub(acc[s], seg[s]);
            else acc[s] = (jb[s] == 0) ? seg[s] : rn_add(acc[s], seg[s]);
            seg[s] = 0.0;
        };
        auto loadx = [&](int32_t c, double (&xs)[KZ]) {
            // one IMAD.WIDE.U32: base + c * (8 D) bytes (offsets < 2^32 bytes)
            const double *xp = reinterpret_cast<const double *>(reinterpret_cast<const char *>(xb) +
                                                                (uint64_t)(uint32_t)c * (uint32_t)D8);
#pragma unroll
            for (int s = 0; s < KZ; ++s) {
                if constexpr (W) xs[s] = __ldg(xp + s * 32);
                else xs[s] = zok[s] ? __ldg(xp + s * L) : 0.0;
            }
        };
        auto step = [&](int32_t c, double v, const double (&xs)[KZ]) {
            if constexpr (ALIGNED) {
                while (c >= thr[0]) {
#pragma unroll
                    for (int s = 0; s < KZ; ++s) { fold(s); ++jb[s]; }
                    thr[0] = (int32_t)__ldg(A.sbounds + jb[0] + 1);
                }
            } else {
#pragma unroll
                for (int s = 0; s < KZ; ++s) {
                    while (c >= thr[s]) {
                        fold(s);
                        ++jb[s];
                        thr[s] = (int32_t)((__ldg(A.bounds + jb[s] + 1) - (zb + s * L) + D - 1) / D);
                    }
                }
            }
#pragma unroll
            for (int s = 0; s < KZ; ++s) seg[s] = rn_add(seg[s], rn_mul(v, xs[s]));
        };
        // entries of a row are in ascending stored index: if the last of four
        // is below every threshold, none of them crosses a block bound
        auto below = [&](int32_t c) {
            bool b = c < thr[0];
            if constexpr (!ALIGNED)
#pragma unroll
                for (int s = 1; s < KZ; ++s) b = b && c < thr[s];
            return b;
        };
        const int64_t beg = live ? A.ptr[r] : 0, end = live ? A.ptr[r + 1] : 0;
        int64_t k = beg;
        const int64_t kh = ((beg + 3) & ~(int64_t)3) < end ? ((beg + 3) & ~(int64_t)3) : end;
        for (; k < kh; ++k) {
            const int32_t c = ld_stream(idx + k, pol);
            const double v = (double)ld_stream(val + k, pol);
            double xs[KZ];
            loadx(c, xs);
            step(c, v, xs);
        }
        for (; k + 4 <= end; k += 4) {
            int32_t c[4];
            double v[4], xs[4][KZ];
            stk_load4<V>(idx, val, k, pol, c, v);
#pragma unroll
            for (int u = 0; u < 4; ++u) loadx(c[u], xs[u]);
            if (below(c[3])) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int s = 0; s < KZ; ++s) seg[s] = rn_add(seg[s], rn_mul(v[u], xs[u][s]));
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) step(c[u], v[u], xs[u]);
            }
        }
        for (; k < end; ++k) {
            const int32_t c = ld_stream(idx + k, pol);
            const double v = (double)ld_stream(val + k, pol);
            double xs[KZ];
            loadx(c, xs);
            step(c, v, xs);
        }
#pragma unroll
        for (int s = 0; s < KZ; ++s) {
            if (zok[s]) {
                for (; jb[s] < A.nb; ++jb[s]) fold(s);  // the open segment, then empty trailing blocks
                epi(r * D + zb + s * L, acc[s]);
            }
        }
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.flush(v);
        block_sum<Epi::K>(v, sm);
        if (threadIdx.x == 0 && part != nullptr)
            for (int k = 0; k < Epi::K; ++k) part[(size_t)blockIdx.x * Epi::K + k] = v[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != nullptr) cnt[0] = gridDim.x;
}

// ---------------------------------------------------------------------------
// Tile-staged products.  Stored rows are grouped into tiles of <= 16 rows that
// share most of their columns (4x4 pixel tiles of A2^T: 4.0 entries per
// distinct ray; 4 angles x 4 bins of A2: 3.45 entries per distinct pixel,
// measured at 256^2 x 360 x 363).  Per tile the plan keeps the sorted union of
// the tile's columns and, per entry, its position in that union (uint16, rows
// padded to multiples of 4 with a sentinel).  A CTA takes one (tile, slice
// chunk): the vector rows of the union stream through a double-buffered
// shared-memory window with cp.async (one global read per distinct column
// instead of one per entry), and 16 lanes per tile row accumulate from shared
// memory.  Entries are still consumed in the row's stored order, so every
// output keeps the exact block-sequential arithmetic of the kernel above.
// ---------------------------------------------------------------------------
struct StkTiles {
    int64_t ntiles;
    const int64_t *tile_ptr;   // [ntiles + 1] -> tile rows
    const int32_t *tile_rows;  // stored row id of each tile row
    const int64_t *row_ptr;    // [tile rows + 1] entry ranges, multiples of 4
    const uint16_t *loc;       // position of the entry's column in the tile union; 0xFFFF = padding
    const void *val;           // entry values (V), 0 for padding
    const int64_t *uni_ptr;    // [ntiles + 1]
    const int32_t *uni;        // sorted distinct stored columns per tile
};

constexpr int kTileRows = 16;   // rows per tile (one per 16-lane group)
constexpr int kTileSeg = 64;    // union columns per shared-memory window

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int KZ>
constexpr size_t stk_tile_smem() {
    return sizeof(double) * 2 * kTileSeg * 16 * KZ + sizeof(int32_t) * 2 * kTileSeg;
}

template <typename V, int KZ, bool RESID, bool ALIGNED, class Epi>
__global__ void __launch_bounds__(kThreads, 2) stacked_tile_kernel(Stk<V> A, StkTiles T, Epi epi, double *part,
                                                                    int64_t *cnt) {
    constexpr int ZC = 16 * KZ;
    extern __shared__ double win[];                    // [2][kTileSeg][ZC]
    int32_t *wcol = reinterpret_cast<int32_t *>(win + 2 * kTileSeg * ZC);  // [2][kTileSeg]
    __shared__ double sm[8 * (kThreads / 32)];
    const int tr = threadIdx.x >> 4, lane = threadIdx.x & 15;
    const int32_t D = (int32_t)A.D;
    const int64_t nchunks = D / ZC;
    const int64_t items = T.ntiles * nchunks;
    const uint64_t pol = policy_evict_first();
    const V *__restrict__ val = reinterpret_cast<const V *>(T.val);

    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t ch = it / T.ntiles, t = it - ch * T.ntiles;
        const int32_t z0 = (int32_t)ch * ZC;
        const int64_t r0 = T.tile_ptr[t], nr = T.tile_ptr[t + 1] - r0;
        const int64_t u0 = T.uni_ptr[t];
        const int nu = (int)(T.uni_ptr[t + 1] - u0);
        const bool live = tr < nr;
        const int64_t srow = live ? T.tile_rows[r0 + tr] : 0;
        int64_t e = live ? T.row_ptr[r0 + tr] : 0;
        const int64_t e_end = live ? T.row_ptr[r0 + tr + 1] : 0;
        double seg[KZ], acc[KZ];
        int32_t thr[KZ];
        int jb[KZ];
#pragma unroll
        for (int s = 0; s < KZ; ++s) {
            const int32_t z = z0 + lane + 16 * s;
            seg[s] = 0.0;
            acc[s] = (RESID && live) ? A.y[srow * D + z] : 0.0;
            jb[s] = 0;
            if constexpr (ALIGNED) thr[s] = (int32_t)__ldg(A.sbounds + 1);
            else thr[s] = (int32_t)((__ldg(A.bounds + 1) - z + D - 1) / D);
        }
        auto fold = [&](int s) {
            if constexpr (RESID) acc[s] = rn_sub(acc[s], seg[s]);
            else acc[s] = (jb[s] == 0) ? seg[s] : rn_add(acc[s], seg[s]);
            seg[s] = 0.0;
        };
        // stage union columns [j0, j0 + kTileSeg) of the vector chunk into buffer b
        auto stage = [&](int j0, int b) {
            const int nj = (nu - j0) < kTileSeg ? (nu - j0) : kTileSeg;
            constexpr int PER = ZC / 2;  // 16-byte pieces per union column
            for (int q = threadIdx.x; q < nj * PER; q += kThreads) {
                const int j = q / PER, piece = q - j * PER;
                const int32_t col = __ldg(T.uni + u0 + j0 + j);
                cp_async16(win + ((size_t)b * kTileSeg + j) * ZC + 2 * piece, A.vec + (int64_t)col * D + z0 + 2 * piece);
            }
            for (int j = threadIdx.x; j < nj; j += kThreads) wcol[b * kTileSeg + j] = __ldg(T.uni + u0 + j0 + j);
            cp_async_commit();
        };
        const int nseg = (nu + kTileSeg - 1) / kTileSeg;
        // entry cursor: 4 entries at a time (rows are padded to multiples of 4)
        uint16_t lb[4] = {0xFFFF, 0xFFFF, 0xFFFF, 0xFFFF};
        double vb[4] = {0.0, 0.0, 0.0, 0.0};
        int pos = 4;
        auto refill = [&]() {
            const uint2 l2 = __ldg(reinterpret_cast<const uint2 *>(T.loc + e));
            lb[0] = (uint16_t)(l2.x & 0xFFFF); lb[1] = (uint16_t)(l2.x >> 16);
            lb[2] = (uint16_t)(l2.y & 0xFFFF); lb[3] = (uint16_t)(l2.y >> 16);
            if constexpr (sizeof(V) == 4) {
                const float4 v4 = ld_stream4(reinterpret_cast<const float *>(val) + e, pol);
                vb[0] = v4.x; vb[1] = v4.y; vb[2] = v4.z; vb[3] = v4.w;
            } else {
                const double2 a2 = ld_stream2(reinterpret_cast<const double *>(val) + e, pol);
                const double2 b2 = ld_stream2(reinterpret_cast<const double *>(val) + e + 2, pol);
                vb[0] = a2.x; vb[1] = a2.y; vb[2] = b2.x; vb[3] = b2.y;
            }
            e += 4;
            pos = 0;
        };
        if (nseg > 0) stage(0, 0);
        for (int sg = 0; sg < nseg; ++sg) {
            const int b = sg & 1;
            if (sg + 1 < nseg) {
                stage((sg + 1) * kTileSeg, b ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const int j0 = sg * kTileSeg;
            const int jend = j0 + kTileSeg;
            const double *wb = win + (size_t)b * kTileSeg * ZC + lane;
            const int32_t *cb = wcol + b * kTileSeg;
            if (live) {
                for (;;) {
                    if (pos == 4) {
                        if (e >= e_end) break;
                        refill();
                    }
                    int done = 4;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (u >= pos && done == 4) {
                            const int l = lb[u];
                            if (l >= jend) {
                                done = u;
                            } else {
                                const int jl = l - j0;
                                const int32_t c = cb[jl];
                                if constexpr (ALIGNED) {
                                    while (c >= thr[0]) {
#pragma unroll
                                        for (int s = 0; s < KZ; ++s) { fold(s); ++jb[s]; }
                                        thr[0] = (int32_t)__ldg(A.sbounds + jb[0] + 1);
                                    }
                                } else {
#pragma unroll
                                    for (int s = 0; s < KZ; ++s) {
                                        while (c >= thr[s]) {
                                            fold(s);
                                            ++jb[s];
                                            thr[s] = (int32_t)((__ldg(A.bounds + jb[s] + 1) - (z0 + lane + 16 * s) + D - 1) / D);
                                        }
                                    }
                                }
                                const double v = vb[u];
#pragma unroll
                                for (int s = 0; s < KZ; ++s) seg[s] = rn_add(seg[s], rn_mul(v, wb[jl * ZC + 16 * s]));
                            }
                        }
                    }
                    if (done < 4) { pos = done; break; }
                    pos = 4;
                }
            }
            __syncthreads();  // buffer b is restaged two windows later
        }
        if (live) {
#pragma unroll
            for (int s = 0; s < KZ; ++s) {
                for (; jb[s] < A.nb; ++jb[s]) fold(s);
                epi(srow * D + z0 + lane + 16 * s, acc[s]);
            }
        }
    }
    if constexpr (Epi::K > 0) {
        double v[Epi::K];
        epi.flush(v);
        block_sum<Epi::K>(v, sm);
        if (threadIdx.x == 0 && part != nullptr)
            for (int k = 0; k < Epi::K; ++k) part[(size_t)blockIdx.x * Epi::K + k] = v[k];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != nullptr) cnt[0] = gridDim.x;
}

// ---------------------------------------------------------------------------
// block-restricted and stochastic-pair products (thread per interleaved output)
// ---------------------------------------------------------------------------

// out[O - o0] = sum over stored row O / D, entries with E = e*D + O%D in [e0, e1):
// A2[.,.] vec[E - e0]   (orc_block_matvec / orc_block_rmatvec order)
template <typename V>
__global__ void __launch_bounds__(kThreads) stacked_block_kernel(const int64_t *ptr, const int32_t *idx,
                                                                 const V *val, int64_t D, int64_t o0,
                                                                 int64_t o1, int64_t e0, int64_t e1,
                                                                 const double *vec, double *out) {
    for (int64_t O = o0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; O < o1;
         O += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = O / D, z = O - r * D;
        double s = 0.0;
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int64_t E = (int64_t)idx[k] * D + z;
            if (E >= e1) break;
            if (E >= e0) s = rn_add(s, rn_mul((double)val[k], vec[E - e0]));
        }
        out[O - o0] = s;
    }
}

// z_cache[j, R] for the selected (row block of R, j) pairs; then r_next[R] =
// y[R] - z_cache[0, R] - ... for every R (solvers.py:274-297, alpha/gamma < 1)
template <typename V>
__global__ void __launch_bounds__(kThreads) stacked_pair_forward_kernel(
    const int64_t *ptr, const int32_t *idx, const V *val, int64_t D, int64_t rows, const int64_t *rb, int64_t M,
    const int64_t *cb, int64_t N, BlockMask rsel, BlockMask csel, const double *x, const double *y,
    double *z_cache, double *r_next) {
    for (int64_t R = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; R < rows; R += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = R / D, z = R - r * D;
        if (rsel.has(block_of(rb, M, R))) {
            int64_t j = 0;
            double s = 0.0;
            for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
                const int64_t C = (int64_t)idx[k] * D + z;
                while (C >= cb[j + 1]) {
                    if (csel.has(j)) z_cache[j * rows + R] = s;
                    s = 0.0;
                    ++j;
                }
                s = rn_add(s, rn_mul((double)val[k], x[C]));
            }
            for (; j < N; ++j) {
                if (csel.has(j)) z_cache[j * rows + R] = s;
                s = 0.0;
            }
        }
        double acc = y[R];
        for (int64_t j = 0; j < N; ++j) acc = rn_sub(acc, z_cache[j * rows + R]);
        r_next[R] = acc;
    }
}

// g[C] = 2 * (0 + t_i1 + t_i2 + ...) over the selected row blocks in ascending
// order for columns of selected column blocks, 0 elsewhere (solvers.py:299-303)
template <typename V>
__global__ void __launch_bounds__(kThreads) stacked_pair_grad_kernel(
    const int64_t *tptr, const int32_t *tidx, const V *tval, int64_t D, int64_t cols, const int64_t *rb, int64_t M,
    const int64_t *cb, int64_t N, BlockMask rsel, BlockMask csel, const double *r, double *g) {
    for (int64_t C = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; C < cols; C += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        if (csel.has(block_of(cb, N, C))) {
            const int64_t c = C / D, z = C - c * D;
            int64_t i = 0;
            double s = 0.0;
            for (int64_t k = tptr[c]; k < tptr[c + 1]; ++k) {
                const int64_t R = (int64_t)tidx[k] * D + z;
                while (R >= rb[i + 1]) {
                    if (rsel.has(i)) acc = rn_add(acc, s);
                    s = 0.0;
                    ++i;
                }
                s = rn_add(s, rn_mul((double)tval[k], r[R]));
            }
            for (; i < M; ++i) {
                if (rsel.has(i)) acc = rn_add(acc, s);
                s = 0.0;
            }
        }
        g[C] = 2.0 * acc;
    }
}

// nnz of every (row block, column block) of A2 (x) I_D; tbl in shared memory
// when M*N <= kStkTbl, else global atomics
constexpr int kStkTbl = 4096;
__global__ void __launch_bounds__(kThreads) stacked_block_nnz_kernel(const int64_t *ptr, const int32_t *idx, int64_t D,
                                                                     int64_t rows, const int64_t *rb, int64_t M,
                                                                     const int64_t *cb, int64_t N,
                                                                     unsigned long long *cnt) {
    __shared__ unsigned long long tbl[kStkTbl];
    const bool local = M * N <= kStkTbl;
    if (local)
        for (int64_t t = threadIdx.x; t < M * N; t += blockDim.x) tbl[t] = 0;
    __syncthreads();
    unsigned long long *dst = local ? tbl : cnt;
    for (int64_t R = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; R < rows; R += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = R / D, z = R - r * D;
        const int64_t i = block_of(rb, M, R);
        int64_t j = 0;
        unsigned long long run = 0;
        for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int64_t C = (int64_t)idx[k] * D + z;
            while (C >= cb[j + 1]) {
                if (run) atomicAdd(dst + i * N + j, run);
                run = 0;
                ++j;
            }
            ++run;
        }
        if (run) atomicAdd(dst + i * N + j, run);
    }
    if (local) {
        __syncthreads();
        for (int64_t t = threadIdx.x; t < M * N; t += blockDim.x)
            if (tbl[t]) atomicAdd(cnt + t, tbl[t]);
    }
}

}  // namespace bsgd
