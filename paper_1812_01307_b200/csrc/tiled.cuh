// Panel-tiled SpMV: vector panels in shared memory, A streamed by TMA.
//
// Why: a random gather through L1 costs one tag-stage slot per distinct
// sector (~1 per SM per cycle, profiles/r01_gather_microbench.md), which caps
// the vector-CSR kernels at ~0.29 ms per configs[1] product, 3.5x above the HBM
// bound.  Gathers from the CTA's own shared memory run ~5x faster.
//
// Layout ("tiles"): rows are cut into groups of R rows, the gathered vector
// into panels of P entries.  Tile (g, p) holds the nonzeros of rows in group g
// and columns in panel p, in CSR order, each packed as (row_local << 16 |
// col_local) plus its value.  Tiles are stored group-major, panel-minor.  Each
// tile is cut into "row chunks" (<= 32 entries and never splitting a row, or
// one long row) and row chunks are packed into "units" of <= CH entries, the
// granule a TMA bulk copy moves.
//
// Kernel (one CTA per SM, clusters of CL CTAs, each CTA owns one row group at
// a time; all CTAs of a cluster walk the panels in lockstep):
//   warp 0  ring producer: TMA-copies the CTA's units into an NS-slot ring;
//   warp 1  panel producer: the cluster leader multicasts vector panel p into
//           every member's double buffer once all members released it, so
//           each panel is read from L2 once per cluster;
//   warps 2+ consumers: per row chunk, gather vec from the smem panel, reduce
//           the row segments with a shuffle scan, add into a shared-memory
//           row accumulator (each row once per tile -> deterministic), and
//           finally run the same epilogue functors as the CSR kernels.
#pragma once

#include "common.cuh"
#include "sm100.cuh"

namespace bsgd {

constexpr int kTileConsumerWarps = 16;
constexpr int kTileThreads = 32 * (2 + kTileConsumerWarps);
constexpr int kTileCL = 8;     // cluster size (portable)
constexpr int kTileNS = 3;     // ring slots
constexpr int kTileMaxNP = 1023;

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
    const uint32_t *unit_rc;      // [NU+1] row-chunk index range
    const uint16_t *rc_off;       // [NRC+8] chunk start within its unit
    const uint32_t *tile_unit;    // [NG*NP+1] unit range of each tile
    const double *vec;            // gathered vector, ncols
};

// per-slot unit descriptor written by the ring producer into shared memory
struct UnitMeta {
    uint32_t len;      // entries in the unit
    uint32_t kdelta;   // first entry's offset inside the slot (copy starts 16-byte aligned)
    uint32_t nrc;      // row chunks
    uint32_t rdelta;   // first chunk offset's index inside the slot's rc area
};

template <typename V>
struct TileSmem {
    static constexpr int CH = TileCfg<V>::CH;
    static constexpr int SLOT = CH + 8;       // + alignment slack (copies start at a 4-entry boundary)
    static constexpr int RCSLOT = CH + 16;    // u16 chunk offsets + 8-entry alignment slack
    static size_t bytes(int R, int P) {
        size_t b = 0;
        b += (size_t)2 * P * sizeof(double);                 // vector panels
        b += (size_t)kTileNS * SLOT * sizeof(uint32_t);      // ring keys
        b += (size_t)kTileNS * SLOT * sizeof(V);             // ring values
        b += (size_t)kTileNS * RCSLOT * sizeof(uint16_t);    // ring chunk offsets
        b += (size_t)kTileNS * sizeof(UnitMeta);             // ring unit descriptors
        b += (size_t)R * sizeof(double);                     // row accumulators
        b += (size_t)(kTileMaxNP + 1) * sizeof(uint32_t);    // tile -> unit range of the group
        b += 16 * sizeof(uint64_t);                          // barriers
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
        packed[k] = ((uint32_t)(r % R) << 16) | (uint32_t)(c % P);
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

// Greedy row-chunk / unit segmentation of one tile (sequential per tile).
// Pass 0 counts (n_rc[t], n_unit[t]); pass 1 writes at the scanned offsets.
// bad |= 1 if a row has more than CH entries inside one tile.
template <int CH>
__global__ void tile_segment_kernel(int64_t ntiles, const uint64_t *tile_ptr, const uint32_t *keys, int pass,
                                    uint32_t *n_rc, uint32_t *n_unit, const uint32_t *rc_base,
                                    const uint32_t *unit_base, uint64_t *unit_start, uint32_t *unit_len,
                                    uint32_t *unit_rc, uint16_t *rc_off, int *bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t t0 = tile_ptr[t], t1 = tile_ptr[t + 1];
        uint32_t rc = 0, un = 0;
        const uint32_t rcb = pass ? rc_base[t] : 0, unb = pass ? unit_base[t] : 0;
        uint64_t us = t0;      // current unit start
        uint64_t ulen = 0;     // current unit length
        uint64_t cs = t0;      // current chunk start
        uint64_t i = t0;
        auto emit_chunk = [&](uint64_t a, uint64_t b) {
            if (ulen > 0 && ulen + (b - a) > (uint64_t)CH) {  // close the unit
                if (pass) { unit_start[unb + un] = us; unit_len[unb + un] = (uint32_t)ulen; }
                ++un;
                ulen = 0;
            }
            if (ulen == 0) {
                us = a;
                if (pass) unit_rc[unb + un] = rcb + rc;
            }
            if (pass) rc_off[rcb + rc] = (uint16_t)(a - us);
            ++rc;
            ulen = b - us;
        };
        while (i < t1) {
            const uint32_t row = keys[i] >> 16;
            uint64_t j = i + 1;
            while (j < t1 && (keys[j] >> 16) == row) ++j;
            const uint64_t rl = j - i;
            if (rl > (uint64_t)CH) atomicOr(bad, 1);
            if (rl > 32) {
                if (i > cs) emit_chunk(cs, i);
                emit_chunk(i, j);
                cs = j;
            } else if (i - cs + rl > 32) {
                emit_chunk(cs, i);
                cs = i;
            }
            i = j;
        }
        if (t1 > cs) emit_chunk(cs, t1);
        if (ulen > 0) {
            if (pass) { unit_start[unb + un] = us; unit_len[unb + un] = (uint32_t)ulen; }
            ++un;
        }
        if (!pass) { n_rc[t] = rc; n_unit[t] = un; }
    }
}

__global__ void tile_finish_kernel(int64_t ntiles, const uint32_t *n_unit, const uint32_t *unit_base,
                                   uint32_t total_units, uint32_t total_rc, uint32_t *tile_unit,
                                   uint32_t *unit_rc) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles; t += (int64_t)gridDim.x * blockDim.x) {
        tile_unit[t] = (t < ntiles) ? unit_base[t] : total_units;
        if (t == ntiles) unit_rc[total_units] = total_rc;
    }
    (void)n_unit;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <typename V, class Epi>
__global__ void __launch_bounds__(kTileThreads, 1) tile_spmv_kernel(Tiled<V> T, Epi epi, double *part, int64_t *cnt) {
    constexpr int SLOT = TileSmem<V>::SLOT;
    constexpr int RCSLOT = TileSmem<V>::RCSLOT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *xbuf = reinterpret_cast<double *>(smem_raw);                              // [2][P]
    uint32_t *rkeys = reinterpret_cast<uint32_t *>(xbuf + 2 * (size_t)T.P);           // [NS][SLOT]
    V *rvals = reinterpret_cast<V *>(rkeys + (size_t)kTileNS * SLOT);                 // [NS][SLOT]
    uint16_t *rrc = reinterpret_cast<uint16_t *>(rvals + (size_t)kTileNS * SLOT);     // [NS][RCSLOT]
    UnitMeta *rmeta = reinterpret_cast<UnitMeta *>(rrc + (size_t)kTileNS * RCSLOT);   // [NS]
    double *acc = reinterpret_cast<double *>(rmeta + kTileNS);                        // [R]
    uint32_t *tu = reinterpret_cast<uint32_t *>(acc + T.R);                           // [NP+1]
    uint64_t *bars = reinterpret_cast<uint64_t *>(tu + kTileMaxNP + 1);
    uint64_t *ring_full = bars;            // [NS]
    uint64_t *ring_empty = bars + 4;       // [NS]
    uint64_t *x_full = bars + 8;           // [2]
    uint64_t *x_free = bars + 10;          // [2] this CTA's consumers released the slot
    uint64_t *x_clus = bars + 12;          // [2] (leader) all cluster members released the slot

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t ncl = num_clusters();
    const uint32_t cid = cluster_id();
    const int64_t ctas = (int64_t)ncl * kTileCL;
    const int64_t my = (int64_t)cid * kTileCL + rank;
    const int rounds = (int)((T.NG + ctas - 1) / ctas);
    const int P = T.P, NP = T.NP;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTileNS; ++s) { mbar_init(ring_full + s, 1); mbar_init(ring_empty + s, 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(x_full + s, 1); mbar_init(x_free + s, 1); mbar_init(x_clus + s, kTileCL); }
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();

    if (warp == 0) {
        // ---------------- ring producer (whole warp: metadata is fetched 32 units at a time) ----------------
        uint32_t k = 0;
        for (int rd = 0; rd < rounds; ++rd) {
            const int64_t g = my + (int64_t)rd * ctas;
            if (g >= T.NG) continue;
            const uint32_t u0 = T.tile_unit[g * NP], u1 = T.tile_unit[(g + 1) * NP];
            for (uint32_t ub = u0; ub < u1; ub += 32) {
                const uint32_t u = ub + lane;
                uint64_t m_st = 0;
                uint32_t m_len = 0, m_r0 = 0, m_r1 = 0;
                if (u < u1) { m_st = T.unit_start[u]; m_len = T.unit_len[u]; m_r0 = T.unit_rc[u]; m_r1 = T.unit_rc[u + 1]; }
                const uint32_t nb = (u1 - ub < 32u) ? (u1 - ub) : 32u;
                for (uint32_t j = 0; j < nb; ++j, ++k) {
                    const uint64_t st = __shfl_sync(0xffffffffu, m_st, j);
                    const uint32_t len = __shfl_sync(0xffffffffu, m_len, j);
                    const uint32_t r0 = __shfl_sync(0xffffffffu, m_r0, j);
                    const uint32_t r1 = __shfl_sync(0xffffffffu, m_r1, j);
                    if (lane == 0) {
                        const int s = k % kTileNS;
                        if (k >= (uint32_t)kTileNS) mbar_wait(ring_empty + s, ((k / kTileNS) - 1) & 1);
                        const uint64_t a0 = st & ~(uint64_t)3;
                        const uint64_t a1 = (st + len + 3) & ~(uint64_t)3;
                        const uint32_t n4 = (uint32_t)(a1 - a0);
                        const uint32_t c0 = r0 & ~7u, c1 = (r1 + 7u) & ~7u;
                        const uint32_t nrc8 = c1 - c0;
                        UnitMeta m;
                        m.len = len; m.kdelta = (uint32_t)(st - a0); m.nrc = r1 - r0; m.rdelta = r0 - c0;
                        rmeta[s] = m;
                        mbar_arrive_expect_tx(ring_full + s,
                                              n4 * (uint32_t)(sizeof(uint32_t) + sizeof(V)) + nrc8 * 2u);
                        bulk_g2s(rkeys + (size_t)s * SLOT, T.keys + a0, n4 * sizeof(uint32_t), ring_full + s);
                        bulk_g2s(rvals + (size_t)s * SLOT, T.vals + a0, n4 * (uint32_t)sizeof(V), ring_full + s);
                        bulk_g2s(rrc + (size_t)s * RCSLOT, T.rc_off + c0, nrc8 * 2u, ring_full + s);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- vector-panel producer (lockstep across the cluster) ----------------
        if (lane == 0) {
            const int total = rounds * NP;
            for (int q = 0; q < total; ++q) {
                const int s = q & 1;
                const int p = q % NP;
                const int64_t c0 = (int64_t)p * P;
                const int64_t n = (T.ncols - c0 < P) ? (T.ncols - c0) : P;
                const uint32_t bytes = (uint32_t)((n & ~(int64_t)1) * sizeof(double));
                if (q >= 2) mbar_wait(x_free + s, ((q >> 1) - 1) & 1);
                mbar_arrive_expect_tx(x_full + s, bytes);
                mbar_arrive_remote(x_clus + s, 0);
                if (rank == 0) {
                    mbar_wait_cluster(x_clus + s, (q >> 1) & 1);
                    if (bytes > 0)
                        bulk_g2s_multicast(xbuf + (size_t)s * P, T.vec + c0, bytes, x_full + s,
                                           (uint16_t)((1u << kTileCL) - 1));
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- consumers ----------------
        const int cw = warp - 2;
        const int ctid = threadIdx.x - 64;
        constexpr uint32_t NCT = 32 * kTileConsumerWarps;
        uint32_t k = 0;   // unit counter (matches the producer)
        int q = 0;        // panel counter
        for (int rd = 0; rd < rounds; ++rd) {
            const int64_t g = my + (int64_t)rd * ctas;
            const bool live = g < T.NG;
            for (int i = ctid; i < T.R; i += NCT) acc[i] = 0.0;
            if (live)
                for (int i = ctid; i <= NP; i += NCT) tu[i] = T.tile_unit[g * NP + i];
            named_bar_sync(1, NCT);
            for (int p = 0; p < NP; ++p, ++q) {
                const int s = q & 1;
                mbar_wait(x_full + s, (q >> 1) & 1);
                const double *xs = xbuf + (size_t)s * P;
                const int64_t c0 = (int64_t)p * P;
                const int64_t n = (T.ncols - c0 < P) ? (T.ncols - c0) : P;
                if (n & 1) {  // odd tail element is not covered by the 16-byte bulk copy
                    if (ctid == 0) {
                        xbuf[(size_t)s * P + n - 1] = T.vec[c0 + n - 1];
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    named_bar_sync(1, NCT);
                }
                if (live) {
                    const uint32_t u0 = tu[p], u1 = tu[p + 1];
                    for (uint32_t u = u0; u < u1; ++u, ++k) {
                        const int rs = k % kTileNS;
                        mbar_wait(ring_full + rs, (k / kTileNS) & 1);
                        const UnitMeta m = rmeta[rs];
                        const uint32_t *kk = rkeys + (size_t)rs * SLOT + m.kdelta;
                        const V *vv = rvals + (size_t)rs * SLOT + m.kdelta;
                        const uint16_t *ro = rrc + (size_t)rs * RCSLOT + m.rdelta;
                        for (uint32_t rc = cw; rc < m.nrc; rc += kTileConsumerWarps) {
                            const uint32_t e0 = ro[rc];
                            const uint32_t e1 = (rc + 1 < m.nrc) ? ro[rc + 1] : m.len;
                            const uint32_t nn = e1 - e0;
                            if (nn <= 32) {
                                const bool valid = lane < (int)nn;
                                const uint32_t key = valid ? kk[e0 + lane] : 0u;
                                const int row = valid ? (int)(key >> 16) : -1 - lane;
                                const int rp = __shfl_up_sync(0xffffffffu, row, 1);
                                const bool head = valid && (lane == 0 || rp != row);
                                const uint32_t heads = __ballot_sync(0xffffffffu, head);
                                const int nseg = __popc(heads);
                                if (nseg > 4) {
                                    // one lane per row: sequential left-to-right sum of its entries
                                    if (lane < nseg) {
                                        const int b = __fns(heads, 0, lane + 1);
                                        const int e = (lane + 1 < nseg) ? __fns(heads, 0, lane + 2) : (int)nn;
                                        const uint32_t k0 = kk[e0 + b];
                                        double v = (double)vv[e0 + b] * xs[k0 & 0xFFFFu];
                                        for (int t = b + 1; t < e; ++t) {
                                            const uint32_t kt = kk[e0 + t];
                                            v = fma((double)vv[e0 + t], xs[kt & 0xFFFFu], v);
                                        }
                                        acc[k0 >> 16] += v;
                                    }
                                } else {
                                    double v = valid ? (double)vv[e0 + lane] * xs[key & 0xFFFFu] : 0.0;
#pragma unroll
                                    for (int off = 1; off < 32; off <<= 1) {
                                        const double vo = __shfl_up_sync(0xffffffffu, v, off);
                                        const int rw = __shfl_up_sync(0xffffffffu, row, off);
                                        if (lane >= off && rw == row) v += vo;
                                    }
                                    const int rn = __shfl_down_sync(0xffffffffu, row, 1);
                                    if (valid && (lane == (int)nn - 1 || rn != row)) acc[row] += v;
                                }
                            } else {  // one long row
                                const uint32_t row = kk[e0] >> 16;
                                double v = 0.0;
                                for (uint32_t e = e0 + lane; e < e1; e += 32)
                                    v = fma((double)vv[e], xs[kk[e] & 0xFFFFu], v);
                                v = warp_sum(v);
                                if (lane == 0) acc[row] += v;
                            }
                        }
                        named_bar_sync(1, NCT);
                        if (ctid == 0) mbar_arrive(ring_empty + rs);
                    }
                }
                named_bar_sync(1, NCT);
                if (ctid == 0) mbar_arrive(x_free + s);
            }
            if (live) {
                const int64_t rbase = g * (int64_t)T.R;
                const int64_t rend = (rbase + T.R < T.nrows) ? rbase + T.R : T.nrows;
                for (int64_t rr = rbase + ctid; rr < rend; rr += NCT) epi(rr, acc[rr - rbase]);
            }
            named_bar_sync(1, NCT);
        }
    }
    __syncwarp();
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
    __syncthreads();
    cluster_sync_all();
}

}  // namespace bsgd
