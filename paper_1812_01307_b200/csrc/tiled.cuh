// Panel-tiled SpMV: vector panels in shared memory, A streamed by TMA.
//
// Why: a random gather through L1 costs one tag-stage slot per distinct
// sector (~1 per SM per cycle, profiles/r01_gather_microbench.md), which caps
// the vector-CSR kernels at ~0.29 ms per configs[1] product, 3.5x above the HBM
// bound.  Gathers from the CTA's own shared memory run ~5x faster.
//
// Layout ("tiles"): rows are cut into groups of R <= 8192 rows, the gathered
// vector into panels of P <= 4096 entries.  Tile (g, p) holds the nonzeros of
// rows in group g and columns in panel p, in CSR order, each packed as
//   key = END << 31 | START << 30 | row_local << 12 | col_local
// (START / END mark the first / last entry of a row inside the tile) plus its
// value.  Tiles are stored group-major, panel-minor and cut into "units" of
// <= CH entries at row boundaries, the granule a TMA bulk copy moves.
//
// Kernel (one persistent CTA per SM).  A work item is (row group g, panel
// range h of H): the CTA streams the tiles (g, p) for p in range h.
//   warp 0  ring producer: TMA-copies the item's units (entries + row-chunk
//           offsets) into an NS-slot ring, unit metadata prefetched 32 at a time;
//   warp 1  panel producer: TMA-copies vector panel p into an NX-slot buffer
//           (per CTA: ~21 TB/s aggregate L2->SM, profiles/r01_gather_microbench.md;
//           a lockstep cluster multicast was measured 2-5x slower per step);
//   warps 2+ consumers: per row chunk, gather the vector from the smem panel,
//           reduce row segments (one lane per row, or a shuffle scan for few
//           rows), add into a shared-memory row accumulator (each row once per
//           tile -> deterministic).  H == 1: the epilogue functor runs here;
//           H > 1: partial sums go to a [H][rows] buffer and a combine kernel
//           adds them in ascending h and runs the epilogue (deterministic).
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace bsgd {

constexpr int kTileConsumerWarps = 30;
constexpr int kTileThreads = 32 * (2 + kTileConsumerWarps);
constexpr int kTileNS = 3;     // ring slots
constexpr int kTileNX = 3;     // vector panel slots
constexpr int kTileMaxNP = 1023;
constexpr int kTileMaxR = 8192;
constexpr int kTileMaxP = 4096;
constexpr int kSplitStride = 32;   // u16 per unit: kTileConsumerWarps + 1 used, padded to 64 bytes
constexpr uint32_t kKeyStart = 1u << 30;
constexpr uint32_t kKeyEnd = 1u << 31;
__host__ __device__ __forceinline__ uint32_t key_row(uint32_t k) { return (k >> 12) & 0x1FFFu; }
__host__ __device__ __forceinline__ uint32_t key_col(uint32_t k) { return k & 0xFFFu; }

template <typename V>
struct TileCfg {
    static constexpr int CH = sizeof(V) == 4 ? 2048 : 1024;  // entries per unit (max)
};

template <typename V>
struct Tiled {
    int64_t nrows, ncols;
    int R, P, NG, NP;
    const uint32_t *keys;
    const V *vals;
    const uint64_t *unit_start;   // [NU]   absolute entry index
    const uint32_t *unit_len;     // [NU]
    const uint16_t *unit_split;   // [NU][kSplitStride] per-consumer-warp entry split points
    const uint32_t *tile_unit;    // [NG*NP+1] unit range of each tile
    const double *vec;            // gathered vector, ncols
    int H;                        // panel ranges per row group (work items = NG * H)
    double *pout;                 // [H][nrows] partial sums when H > 1
};

// per-slot unit descriptor written by the ring producer into shared memory
struct UnitMeta {
    uint32_t len;      // entries in the unit
    uint32_t kdelta;   // first entry's offset inside the slot (copy starts 16-byte aligned)
};
// consumer warp w owns local rows [w*R/16, (w+1)*R/16) of the row group; a
// unit's entries for those rows are [split[w], split[w+1]) (rows are sorted)

template <typename V>
struct TileSmem {
    static constexpr int CH = TileCfg<V>::CH;
    static constexpr int SLOT = CH + 8;       // + alignment slack (copies start at a 4-entry boundary)
    static size_t bytes(int R, int P) {
        size_t b = 0;
        b += (size_t)kTileNX * P * sizeof(double);           // vector panels
        b += (size_t)kTileNS * SLOT * sizeof(uint32_t);      // ring keys
        b += (size_t)kTileNS * SLOT * sizeof(V);             // ring values
        b += (size_t)kTileNS * kSplitStride * sizeof(uint16_t); // ring split points
        b += (size_t)kTileNS * sizeof(UnitMeta);             // ring unit descriptors
        b += (size_t)R * sizeof(double);                     // row accumulators
        b += (size_t)(kTileMaxNP + 1) * sizeof(uint32_t);    // tile -> unit range of the group
        b += 16 * sizeof(uint64_t);                          // barriers (2*NS + 2*NX <= 16)
        return b;
    }
};

// ---------------------------------------------------------------------------
// builder kernels
// ---------------------------------------------------------------------------
__global__ void tile_keys_kernel(int64_t nnz, const int32_t *rowid, const int32_t *col, int R, int P, int NP,
                                 uint32_t *tkey, uint32_t *packed, uint32_t *pos) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rowid[k], c = col[k];
        tkey[k] = (uint32_t)(r / R) * (uint32_t)NP + (uint32_t)(c / P);
        packed[k] = ((uint32_t)(r % R) << 12) | (uint32_t)(c % P);
        pos[k] = (uint32_t)k;
    }
}

template <typename V>
__global__ void tile_gather_kernel(int64_t nnz, const uint32_t *perm, const uint32_t *packed_in, const V *val_in,
                                   uint32_t *keys, V *vals) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = perm[k];
        keys[k] = packed_in[p];
        vals[k] = val_in[p];
    }
}

// START / END flags: first / last entry of a row inside its tile
__global__ void tile_flags_kernel(int64_t nnz, const uint32_t *sorted_tkey, uint32_t *keys) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t key = keys[k];
        const bool start = k == 0 || sorted_tkey[k - 1] != sorted_tkey[k] || key_row(keys[k - 1]) != key_row(key);
        const bool end = k == nnz - 1 || sorted_tkey[k + 1] != sorted_tkey[k] || key_row(keys[k + 1]) != key_row(key);
        keys[k] = key | (start ? kKeyStart : 0u) | (end ? kKeyEnd : 0u);
    }
}

__global__ void tile_ptr_kernel(int64_t ntiles, int64_t nnz, const uint32_t *sorted_tkey, uint64_t *tile_ptr) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = lo + ((hi - lo) >> 1);
            if ((int64_t)sorted_tkey[mid] < t) lo = mid + 1; else hi = mid;
        }
        tile_ptr[t] = (uint64_t)lo;
    }
}

// Greedy unit segmentation of one tile (sequential per tile): whole rows are
// packed into units of <= CH entries.  Pass 0 counts units per tile, pass 1
// writes them at the scanned offsets.  bad |= 1 if a row has more than CH
// entries inside one tile (the tiled path is then not used).
template <int CH>
__global__ void tile_segment_kernel(int64_t ntiles, const uint64_t *tile_ptr, const uint32_t *keys, int pass,
                                    uint32_t *n_unit, const uint32_t *unit_base, uint64_t *unit_start,
                                    uint32_t *unit_len, int *bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t t0 = tile_ptr[t], t1 = tile_ptr[t + 1];
        uint32_t un = 0;
        const uint32_t unb = pass ? unit_base[t] : 0;
        uint64_t us = t0, i = t0;
        while (i < t1) {
            uint64_t j = i + 1;
            while (j < t1 && !(keys[j] & kKeyStart)) ++j;   // row run [i, j)
            if (j - i > (uint64_t)CH) atomicOr(bad, 1);
            if (j - us > (uint64_t)CH && i > us) {          // close the unit before this row
                if (pass) { unit_start[unb + un] = us; unit_len[unb + un] = (uint32_t)(i - us); }
                ++un;
                us = i;
            }
            i = j;
        }
        if (t1 > us) {
            if (pass) { unit_start[unb + un] = us; unit_len[unb + un] = (uint32_t)(t1 - us); }
            ++un;
        }
        if (!pass) n_unit[t] = un;
    }
}

// per-unit split points for the consumer warps (rows are sorted inside a unit)
__global__ void tile_split_kernel(int64_t nunits, const uint64_t *unit_start, const uint32_t *unit_len,
                                  const uint32_t *keys, int R, uint16_t *split) {
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nunits; u += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t st = unit_start[u];
        const uint32_t len = unit_len[u];
        const int rw = (R + kTileConsumerWarps - 1) / kTileConsumerWarps;
        for (int w = 0; w <= kTileConsumerWarps; ++w) {
            uint32_t lo = 0, hi = len;
            const uint32_t bound = (uint32_t)(w * rw);
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (key_row(keys[st + mid]) < bound) lo = mid + 1; else hi = mid;
            }
            split[u * kSplitStride + w] = (uint16_t)lo;
        }
        for (int w = kTileConsumerWarps + 1; w < kSplitStride; ++w) split[u * kSplitStride + w] = 0;
    }
}

__global__ void tile_finish_kernel(int64_t ntiles, const uint32_t *unit_base, uint32_t total_units,
                                   uint32_t *tile_unit) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles; t += (int64_t)gridDim.x * blockDim.x)
        tile_unit[t] = (t < ntiles) ? unit_base[t] : total_units;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tile_item_range(int NP, int H, int h, int &p0, int &p1) {
    const int per = (NP + H - 1) / H;
    p0 = h * per;
    p1 = (p0 + per < NP) ? p0 + per : NP;
    if (p0 > NP) p0 = NP;
}

template <typename V, class Epi>
__global__ void __launch_bounds__(kTileThreads, 1) tile_spmv_kernel(Tiled<V> T, Epi epi, double *part, int64_t *cnt) {
    constexpr int SLOT = TileSmem<V>::SLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *xbuf = reinterpret_cast<double *>(smem_raw);                              // [NX][P]
    uint32_t *rkeys = reinterpret_cast<uint32_t *>(xbuf + kTileNX * (size_t)T.P);     // [NS][SLOT]
    V *rvals = reinterpret_cast<V *>(rkeys + (size_t)kTileNS * SLOT);                 // [NS][SLOT]
    uint16_t *rsplit = reinterpret_cast<uint16_t *>(rvals + (size_t)kTileNS * SLOT);  // [NS][kSplitStride]
    UnitMeta *rmeta = reinterpret_cast<UnitMeta *>(rsplit + (size_t)kTileNS * kSplitStride); // [NS]
    double *acc = reinterpret_cast<double *>(rmeta + kTileNS);                        // [R]
    uint32_t *tu = reinterpret_cast<uint32_t *>(acc + T.R);                           // [NP+1]
    uint64_t *bars = reinterpret_cast<uint64_t *>(tu + kTileMaxNP + 1);
    uint64_t *ring_full = bars;                     // [NS]
    uint64_t *ring_empty = bars + kTileNS;          // [NS]
    uint64_t *x_full = bars + 2 * kTileNS;          // [NX]
    uint64_t *x_free = bars + 2 * kTileNS + kTileNX; // [NX]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = T.P, NP = T.NP, H = T.H;
    const int64_t items = (int64_t)T.NG * H;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTileNS; ++s) { mbar_init(ring_full + s, 1); mbar_init(ring_empty + s, kTileConsumerWarps); }
        for (int s = 0; s < kTileNX; ++s) { mbar_init(x_full + s, 1); mbar_init(x_free + s, kTileConsumerWarps); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- ring producer (whole warp: metadata fetched 32 units at a time) ----------------
        uint32_t k = 0;
        for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
            const int64_t g = w / H;
            int p0, p1;
            tile_item_range(NP, H, (int)(w % H), p0, p1);
            const uint32_t u0 = T.tile_unit[g * NP + p0], u1 = T.tile_unit[g * NP + p1];
            for (uint32_t ub = u0; ub < u1; ub += 32) {
                const uint32_t u = ub + lane;
                uint64_t m_st = 0;
                uint32_t m_len = 0;
                if (u < u1) { m_st = T.unit_start[u]; m_len = T.unit_len[u]; }
                const uint32_t nb = (u1 - ub < 32u) ? (u1 - ub) : 32u;
                for (uint32_t j = 0; j < nb; ++j, ++k) {
                    const uint64_t st = __shfl_sync(0xffffffffu, m_st, j);
                    const uint32_t len = __shfl_sync(0xffffffffu, m_len, j);
                    if (lane == 0) {
                        const int s = k % kTileNS;
                        if (k >= (uint32_t)kTileNS) mbar_wait(ring_empty + s, ((k / kTileNS) - 1) & 1);
                        const uint64_t a0 = st & ~(uint64_t)3;
                        const uint64_t a1 = (st + len + 3) & ~(uint64_t)3;
                        const uint32_t n4 = (uint32_t)(a1 - a0);
                        UnitMeta m;
                        m.len = len; m.kdelta = (uint32_t)(st - a0);
                        rmeta[s] = m;
                        mbar_arrive_expect_tx(ring_full + s, n4 * (uint32_t)(sizeof(uint32_t) + sizeof(V)) +
                                                                 kSplitStride * 2u);
                        bulk_g2s(rkeys + (size_t)s * SLOT, T.keys + a0, n4 * sizeof(uint32_t), ring_full + s);
                        bulk_g2s(rvals + (size_t)s * SLOT, T.vals + a0, n4 * (uint32_t)sizeof(V), ring_full + s);
                        bulk_g2s(rsplit + (size_t)s * kSplitStride, T.unit_split + (size_t)(ub + j) * kSplitStride,
                                 kSplitStride * 2u, ring_full + s);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- vector-panel producer ----------------
        if (lane == 0) {
            int q = 0;
            for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
                int p0, p1;
                tile_item_range(NP, H, (int)(w % H), p0, p1);
                for (int p = p0; p < p1; ++p, ++q) {
                    const int s = q % kTileNX;
                    const int64_t c0 = (int64_t)p * P;
                    const int64_t n = (T.ncols - c0 < P) ? (T.ncols - c0) : P;
                    const uint32_t bytes = (uint32_t)((n & ~(int64_t)1) * sizeof(double));
                    if (q >= kTileNX) mbar_wait(x_free + s, ((q / kTileNX) - 1) & 1);
                    mbar_arrive_expect_tx(x_full + s, bytes);
                    if (bytes > 0) bulk_g2s(xbuf + (size_t)s * P, T.vec + c0, bytes, x_full + s);
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- consumers: warp cw owns local rows [cw*RW, (cw+1)*RW) ----------------
        const int cw = warp - 2;
        const int ctid = threadIdx.x - 64;
        constexpr uint32_t NCT = 32 * kTileConsumerWarps;
        const int RW = (T.R + kTileConsumerWarps - 1) / kTileConsumerWarps;
        const int my_lo = cw * RW, my_hi = (my_lo + RW < T.R) ? my_lo + RW : T.R;
        uint32_t k = 0;   // unit counter (matches the ring producer)
        int q = 0;        // panel counter (matches the panel producer)
        for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
            const int64_t g = w / H;
            const int h = (int)(w % H);
            int p0, p1;
            tile_item_range(NP, H, h, p0, p1);
            for (int i = my_lo + lane; i < my_hi; i += 32) acc[i] = 0.0;
            named_bar_sync(1, NCT);   // every warp finished the previous item's tu[] reads
            for (int i = ctid; i <= p1 - p0; i += NCT) tu[i] = T.tile_unit[g * NP + p0 + i];
            named_bar_sync(1, NCT);
            for (int p = p0; p < p1; ++p, ++q) {
                const int s = q % kTileNX;
                mbar_wait(x_full + s, (q / kTileNX) & 1);
                const double *xs = xbuf + (size_t)s * P;
                const int64_t c0 = (int64_t)p * P;
                const int64_t n = (T.ncols - c0 < P) ? (T.ncols - c0) : P;
                // an odd last panel's final entry is not covered by the 16-byte bulk copy
                const uint32_t tail_col = (n & 1) ? (uint32_t)(n - 1) : 0xFFFFFFFFu;
                const double tail_val = (n & 1) ? T.vec[c0 + n - 1] : 0.0;
                const uint32_t u0 = tu[p - p0], u1 = tu[p - p0 + 1];
                for (uint32_t u = u0; u < u1; ++u, ++k) {
                    const int rs = k % kTileNS;
                    mbar_wait(ring_full + rs, (k / kTileNS) & 1);
                    const UnitMeta m = rmeta[rs];
                    const uint32_t *kk = rkeys + (size_t)rs * SLOT + m.kdelta;
                    const V *vv = rvals + (size_t)rs * SLOT + m.kdelta;
                    const uint32_t b0 = rsplit[rs * kSplitStride + cw], b1 = rsplit[rs * kSplitStride + cw + 1];
                    // the lane holding a row's START entry sums the row left to right
                    for (uint32_t e = b0 + lane; e < b1 + ((32u - ((b1 - b0) & 31u)) & 31u); e += 32) {
                        if (e < b1) {
                            uint32_t key = kk[e];
                            if (key & kKeyStart) {
                                const uint32_t row = key_row(key);
                                uint32_t c = key_col(key);
                                double v = (double)vv[e] * (c == tail_col ? tail_val : xs[c]);
                                uint32_t t = e;
                                while (!(key & kKeyEnd)) {
                                    ++t;
                                    key = kk[t];
                                    c = key_col(key);
                                    v = fma((double)vv[t], (c == tail_col ? tail_val : xs[c]), v);
                                }
                                acc[row] += v;
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(ring_empty + rs);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(x_free + s);
            }
            // epilogue for this warp's rows
            const int64_t rbase = g * (int64_t)T.R;
            const int64_t lo = rbase + my_lo;
            const int64_t hi0 = rbase + my_hi;
            const int64_t hi = (hi0 < T.nrows) ? hi0 : T.nrows;
            if (H == 1) {
                for (int64_t rr = lo + lane; rr < hi; rr += 32) epi(rr, acc[rr - rbase]);
            } else {
                double *dst = T.pout + (size_t)h * T.nrows;
                for (int64_t rr = lo + lane; rr < hi; rr += 32) dst[rr] = acc[rr - rbase];
            }
        }
    }
    __syncwarp();
    if (T.H == 1) {
        // statistics of the epilogue (only consumers carry nonzero values)
        if constexpr (Epi::K > 0) {
            __shared__ double red_sm[Epi::K * (kTileThreads / 32)];
            double v[Epi::K];
            epi.flush(v);
            if (warp < 2)
#pragma unroll
                for (int i = 0; i < Epi::K; ++i) v[i] = 0.0;
            block_sum<Epi::K>(v, red_sm);
            if (threadIdx.x == 0 && part != nullptr)
                for (int i = 0; i < Epi::K; ++i) part[(size_t)blockIdx.x * Epi::K + i] = v[i];
        }
        if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != nullptr) cnt[0] = gridDim.x;
    }
}

// H > 1: rows' partial sums added in ascending h, then the epilogue
template <class Epi>
__global__ void __launch_bounds__(kThreads) tile_combine_kernel(int64_t nrows, int H, const double *pout, Epi epi,
                                                                double *part, int64_t *cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        double s = pout[r];
        for (int h = 1; h < H; ++h) s += pout[(size_t)h * nrows + r];
        epi(r, s);
    }
    if constexpr (Epi::K > 0) {
        __shared__ double sm[Epi::K * (kThreads / 32)];
        double v[Epi::K];
        epi.flush(v);
        block_sum<Epi::K>(v, sm);
        if (threadIdx.x == 0 && part != nullptr)
            for (int i = 0; i < Epi::K; ++i) part[(size_t)blockIdx.x * Epi::K + i] = v[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && cnt != nullptr) cnt[0] = gridDim.x;
}

}  // namespace bsgd
