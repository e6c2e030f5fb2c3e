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
#include "sm100.cuh"

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
// the tile's columns cut into segments of tile_seg<KZ>() columns, and per segment the
// tile rows' entries that fall in it (row-major, uint8 position in the segment
// + value).  Warp-specialised CTA: four producer warps walk the CTA's stream
// of (tile, 128-slice chunk, segment) stages and fill a tile_stages()-deep ring
// with TMA bulk copies -- one 1 KB vector row per distinct column (instead of
// one gather per entry), the entry records, the row offsets -- completing on a
// full-barrier per slot; sixteen consumer warps (one tile row each, four
// slices per lane) accumulate from shared memory and release the slot on an
// empty-barrier.  Each row still consumes its entries in stored order, so every
// output keeps the exact block-sequential arithmetic of the direct kernel.
// ---------------------------------------------------------------------------
constexpr int kTileRows = 16;      // rows per tile
// KZ slices per consumer lane (4, or 8 when the depth is a multiple of 256):
// items of 32 KZ slices, segments of tile_seg<KZ>() columns, so a stage's vector
// window is 32 KB either way and the entry decode is shared by KZ slices
template <int KZ>
__host__ __device__ constexpr int tile_seg() { return KZ == 8 ? 16 : 32; }
template <int KZ>
__host__ __device__ constexpr int tile_zc() { return 32 * KZ; }
// Producer warps: producer p issues ring positions p, p + P, ...; before reusing a
// slot it waits for the slot's previous round on the empty barrier by phase
// parity, which is only unambiguous while no producer can run two rounds ahead
// of the consumers -- guaranteed for P <= the ring depth.
constexpr int kTileProducers = 4;
constexpr int kStkTileThreads = 32 * (16 + kTileProducers);  // 16 consumer warps (one tile row each) + producers

struct StkTiles {
    int64_t ntiles;
    const int64_t *tile_ptr;   // [ntiles + 1] -> tile rows
    const int32_t *tile_rows;  // stored row id of each tile row
    const int64_t *seg_ptr;    // [ntiles + 1] -> segments (>= 1 per tile)
    const int32_t *seg_nj;     // [segments] columns in the segment
    const int64_t *seg_ent;    // [segments] first entry (multiple of 16)
    const uint16_t *seg_row;   // [segments][24] cumulative entry counts per tile row ([16] = total, padded)
    const int32_t *uni;        // [segments][tile_seg] distinct stored columns, per tile ascending (padded)
    const void *ent;           // TileEnt<V> records, per segment padded to 16
};

// one entry: value and (stored column << 8 | position in the segment), one
// shared-memory read per entry
template <typename V>
struct alignas(sizeof(V) == 4 ? 8 : 16) TileEnt {
    V val;
    uint32_t cl;
};

template <typename V, int KZ>
struct TileStage {
    static constexpr size_t win = sizeof(double) * tile_seg<KZ>() * tile_zc<KZ>();
    static constexpr size_t ent = sizeof(TileEnt<V>) * kTileRows * tile_seg<KZ>();
    static constexpr size_t row = 48;
    static constexpr size_t bytes = win + ent + row;
};

// ring depth: as many stages as fit 227 KB of shared memory per CTA
template <typename V, int KZ>
__host__ __device__ constexpr int tile_stages() { return (int)((227 * 1024 - 2048) / TileStage<V, KZ>::bytes); }

template <typename V, int KZ>
__host__ __device__ constexpr size_t stk_tile_smem() {
    return TileStage<V, KZ>::bytes * tile_stages<V, KZ>() + 2 * tile_stages<V, KZ>() * sizeof(uint64_t);
}
static_assert(kTileProducers <= tile_stages<double, 4>() && kTileProducers <= tile_stages<double, 8>(),
              "producers must not outnumber the ring slots");

// Producer warps of the tile-staged kernels: walk the CTA's stream of (tile,
// slice chunk, segment) stages and fill the ring with TMA bulk copies -- one
// vector row per distinct column, the stage's entry records (REC, `hdr` = the
// header slot holding their count, padded to a multiple of `pad`), the header.
template <typename V, class REC, int KZ>
__device__ __forceinline__ void stk_tile_produce(const Stk<V> &A, const StkTiles &T, unsigned char *smraw,
                                                 uint64_t *full, uint64_t *empty, int pw, int hdr, int pad) {
    using ST = TileStage<V, KZ>;
    constexpr int ZC = tile_zc<KZ>();
    constexpr int kTileStages = tile_stages<V, KZ>();
    const int lane = threadIdx.x & 31;
    const int32_t D = (int32_t)A.D;
    const int64_t nchunks = D / ZC;
    const int64_t items = T.ntiles * nchunks;
    auto slot = [&](int k) { return smraw + (size_t)k * ST::bytes; };
    // Segments are issued in batches of four.  A batch's metadata (one
    // segment per lane, shuffled out) and column ids (segment g's ids sit at
    // uni[32 g ..], one per lane) have no dependent loads, and the next
    // batch's are fetched before this batch is issued, so the producer never
    // waits on its own loads.
    constexpr int B = 4;
    int64_t seq = 0;  // stream position of the cursor
    int64_t it = blockIdx.x, g = 0, g1 = 0;
    int32_t z0 = 0;
    auto load_item = [&]() {
        if (it < items) {
            const int64_t t = it % T.ntiles;
            g = T.seg_ptr[t];
            g1 = T.seg_ptr[t + 1];
            z0 = (int32_t)(it / T.ntiles) * ZC;
        }
    };
    load_item();
    struct Batch {
        int64_t gb[B];
        int64_t sq[B];
        int32_t zb[B];
        int nb;
        int64_t m_eb;
        int m_nj, m_ne;
        int32_t col[B];
    };
    auto fetch = [&](Batch &bt) {
        bt.nb = 0;
#pragma unroll
        for (int q = 0; q < B; ++q) {
            bt.gb[q] = -1;
            bt.zb[q] = 0;
            bt.sq[q] = 0;
            // skip the other producers' positions
            while (it < items && seq % kTileProducers != pw) {
                ++seq;
                if (++g == g1) {
                    it += gridDim.x;
                    load_item();
                }
            }
            if (it < items) {
                bt.gb[q] = g;
                bt.zb[q] = z0;
                bt.sq[q] = seq;
                ++bt.nb;
                ++seq;
                if (++g == g1) {
                    it += gridDim.x;
                    load_item();
                }
            }
        }
        int64_t mine = -1;
#pragma unroll
        for (int q = 0; q < B; ++q)
            if (lane == q) mine = bt.gb[q];
        bt.m_eb = 0; bt.m_nj = 0; bt.m_ne = 0;
        if (mine >= 0) {
            bt.m_eb = T.seg_ent[mine];
            bt.m_nj = T.seg_nj[mine];
            bt.m_ne = (T.seg_row[mine * 24 + hdr] + pad - 1) & ~(pad - 1);
        }
#pragma unroll
        for (int q = 0; q < B; ++q)
            bt.col[q] = (bt.gb[q] >= 0 && lane < tile_seg<KZ>()) ? __ldg(T.uni + bt.gb[q] * tile_seg<KZ>() + lane) : 0;
    };
    Batch cur, nxt;
    fetch(cur);
    while (cur.nb > 0) {
        fetch(nxt);
#pragma unroll
        for (int q = 0; q < B; ++q) {
            if (q >= cur.nb) break;
            const int64_t eb = __shfl_sync(0xffffffffu, cur.m_eb, q);
            const int nj = __shfl_sync(0xffffffffu, cur.m_nj, q);
            const int ne = __shfl_sync(0xffffffffu, cur.m_ne, q);
            const int k = (int)(cur.sq[q] % kTileStages);
            const uint32_t round = (uint32_t)(cur.sq[q] / kTileStages);
            if (round > 0) mbar_wait(&empty[k], (round - 1) & 1);
            unsigned char *sb = slot(k);
            const uint32_t bytes = (uint32_t)(nj * ZC * 8 + ne * (int)sizeof(REC) + 48);
            if (lane == 0) mbar_arrive_expect_tx(&full[k], bytes);
            __syncwarp();
            if (lane < nj)
                bulk_g2s(sb + (size_t)lane * ZC * 8, A.vec + (int64_t)cur.col[q] * D + cur.zb[q], ZC * 8, &full[k]);
            if (lane == 1 && ne > 0)
                bulk_g2s(sb + ST::win, reinterpret_cast<const REC *>(T.ent) + eb, ne * sizeof(REC),
                         &full[k]);
            if (lane == 3) bulk_g2s(sb + ST::win + ST::ent, T.seg_row + cur.gb[q] * 24, 48, &full[k]);
            __syncwarp();
        }
        cur = nxt;
    }
}

// slice s of a consumer lane sits at 2 lane + tile_zoff(s) in the stage's 128 slices
__device__ __forceinline__ constexpr int tile_zoff(int s) { return (s & 1) + 64 * (s >> 1); }

// the lane's KZ slice values of one window column (w = column base + 2 lane)
template <int KZ>
__device__ __forceinline__ void tile_xk(const double *w, double (&x)[KZ]) {
#pragma unroll
    for (int m = 0; m < KZ / 2; ++m) {
        const double2 a = *reinterpret_cast<const double2 *>(w + 64 * m);
        x[2 * m] = a.x;
        x[2 * m + 1] = a.y;
    }
}

template <typename V, int KZ, bool RESID, bool ALIGNED, class Epi>
__global__ void __launch_bounds__(kStkTileThreads, 1) stacked_tile_kernel(Stk<V> A, StkTiles T, Epi epi, double *part,
                                                                        int64_t *cnt) {
    using ST = TileStage<V, KZ>;
    constexpr int ZC = tile_zc<KZ>();
    constexpr int kTileStages = tile_stages<V, KZ>();
    extern __shared__ __align__(128) unsigned char smraw[];
    __shared__ double sm[4 * (kStkTileThreads / 32)];
    uint64_t *full = reinterpret_cast<uint64_t *>(smraw + ST::bytes * kTileStages);
    uint64_t *empty = full + kTileStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t D = (int32_t)A.D;
    const int64_t nchunks = D / ZC;
    const int64_t items = T.ntiles * nchunks;
    auto slot = [&](int k) { return smraw + (size_t)k * ST::bytes; };

    if (threadIdx.x == 0) {
        for (int k = 0; k < kTileStages; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], 16);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp >= 16) {
        stk_tile_produce<V, TileEnt<V>, KZ>(A, T, smraw, full, empty, warp - 16, 16, 16);
    } else {
        // ------- consumers: tile row = warp, slices z0 + zoff(lane, s) = 2 lane + (s & 1) + 64 (s >> 1) -------
        // (KZ / 2 16-byte shared-memory reads give a lane its slices, conflict-free)
        constexpr int NH = 1;
        int k = 0;
        uint32_t round = 0;
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
            const int64_t t = it % T.ntiles, ch = it / T.ntiles;
            const int32_t zl = (int32_t)ch * ZC + 2 * lane;
            const int64_t r0 = T.tile_ptr[t], nr = T.tile_ptr[t + 1] - r0;
            const int64_t g0 = T.seg_ptr[t], g1 = T.seg_ptr[t + 1];
            double seg[NH][KZ], acc[NH][KZ];
            int32_t thr[NH][KZ], tmin[NH];
            int jb[NH][KZ];
            int64_t srow[NH];
            bool live[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const int rr = warp + 16 * h;
                live[h] = rr < nr;
                srow[h] = live[h] ? T.tile_rows[r0 + rr] : 0;
#pragma unroll
                for (int s = 0; s < KZ; ++s) {
                    const int32_t z = zl + tile_zoff(s);
                    seg[h][s] = 0.0;
                    acc[h][s] = (RESID && live[h]) ? A.y[srow[h] * D + z] : 0.0;
                    jb[h][s] = 0;
                    if constexpr (ALIGNED) thr[h][s] = (int32_t)__ldg(A.sbounds + 1);
                    else thr[h][s] = (int32_t)((__ldg(A.bounds + 1) - z + D - 1) / D);
                }
                tmin[h] = thr[h][0];
#pragma unroll
                for (int s = 1; s < KZ; ++s) tmin[h] = thr[h][s] < tmin[h] ? thr[h][s] : tmin[h];
            }
            // ALIGNED: every slice crosses the same blocks at the same column, jb[h][0] serves all
            auto fold = [&](int h, int s) {
                if constexpr (RESID) acc[h][s] = rn_sub(acc[h][s], seg[h][s]);
                else acc[h][s] = (jb[h][ALIGNED ? 0 : s] == 0) ? seg[h][s] : rn_add(acc[h][s], seg[h][s]);
                seg[h][s] = 0.0;
            };
            for (int64_t g = g0; g < g1; ++g) {
                mbar_wait(&full[k], round & 1);
                const unsigned char *sb = slot(k);
                const double *w = reinterpret_cast<const double *>(sb) + 2 * lane;
                const TileEnt<V> *ents = reinterpret_cast<const TileEnt<V> *>(sb + ST::win);
                const uint16_t *ro = reinterpret_cast<const uint16_t *>(sb + ST::win + ST::ent);
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    if (!live[h]) continue;
                    const int rr = warp + 16 * h;
                    const int e1 = ro[rr + 1];
                    // block-boundary test of one entry (stored column c), then its products
                    auto cross = [&](int32_t c) {
                        if constexpr (ALIGNED) {
                            while (c >= thr[h][0]) {
#pragma unroll
                                for (int s = 0; s < KZ; ++s) fold(h, s);
                                ++jb[h][0];
                                thr[h][0] = (int32_t)__ldg(A.sbounds + jb[h][0] + 1);
                            }
                            tmin[h] = thr[h][0];
                        } else if (c >= tmin[h]) {
                            // one compare against the smallest threshold guards all slices
#pragma unroll
                            for (int s = 0; s < KZ; ++s) {
                                while (c >= thr[h][s]) {
                                    fold(h, s);
                                    ++jb[h][s];
                                    thr[h][s] = (int32_t)((__ldg(A.bounds + jb[h][s] + 1) - (zl + tile_zoff(s)) + D - 1) / D);
                                }
                            }
                            tmin[h] = thr[h][0];
#pragma unroll
                            for (int s = 1; s < KZ; ++s) tmin[h] = thr[h][s] < tmin[h] ? thr[h][s] : tmin[h];
                        }
                    };
                    int e = ro[rr];
                    // pairs: both entries' shared-memory reads first; entries ascend, so
                    // when the second is below every threshold the first is too
                    for (; e + 1 < e1; e += 2) {
                        const TileEnt<V> r0 = ents[e], r1 = ents[e + 1];
                        const int l0 = r0.cl & 255, l1 = r1.cl & 255;
                        const int32_t c0 = (int32_t)(r0.cl >> 8), c1 = (int32_t)(r1.cl >> 8);
                        const double v0 = (double)r0.val, v1 = (double)r1.val;
                        const double *w0 = w + l0 * ZC, *w1 = w + l1 * ZC;
                        double x0[KZ], x1[KZ];
                        tile_xk<KZ>(w0, x0);
                        tile_xk<KZ>(w1, x1);
                        if (c1 < (ALIGNED ? thr[h][0] : tmin[h])) {
#pragma unroll
                            for (int s = 0; s < KZ; ++s) {
                                seg[h][s] = rn_add(seg[h][s], rn_mul(v0, x0[s]));
                                seg[h][s] = rn_add(seg[h][s], rn_mul(v1, x1[s]));
                            }
                        } else {
                            cross(c0);
#pragma unroll
                            for (int s = 0; s < KZ; ++s) seg[h][s] = rn_add(seg[h][s], rn_mul(v0, x0[s]));
                            cross(c1);
#pragma unroll
                            for (int s = 0; s < KZ; ++s) seg[h][s] = rn_add(seg[h][s], rn_mul(v1, x1[s]));
                        }
                    }
                    if (e < e1) {
                        const TileEnt<V> r = ents[e];
                        const int l = r.cl & 255;
                        cross((int32_t)(r.cl >> 8));
                        const double v = (double)r.val;
                        double xl[KZ];
                        tile_xk<KZ>(w + l * ZC, xl);
#pragma unroll
                        for (int s = 0; s < KZ; ++s) seg[h][s] = rn_add(seg[h][s], rn_mul(v, xl[s]));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[k]);
                if (++k == kTileStages) { k = 0; ++round; }
            }
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                if (!live[h]) continue;
#pragma unroll
                for (int s = 0; s < KZ; ++s) {
                    if constexpr (ALIGNED) {
                        for (int j = jb[h][0]; j < A.nb; ++j) {   // fold's jb test reads jb[h][0]
                            if constexpr (RESID) acc[h][s] = rn_sub(acc[h][s], seg[h][s]);
                            else acc[h][s] = (j == 0) ? seg[h][s] : rn_add(acc[h][s], seg[h][s]);
                            seg[h][s] = 0.0;
                        }
                    } else {
                        for (; jb[h][s] < A.nb; ++jb[h][s]) fold(h, s);
                    }
                    epi(srow[h] * D + zl + tile_zoff(s), acc[h][s]);
                }
            }
        }
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
