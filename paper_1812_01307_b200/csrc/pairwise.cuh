// numpy-order sums on the device.
//
// The reference's TV prox takes every decision from np.sum(...) of a 2-D
// float64 array (tv.py:203,215-216,239-240,251; the fallback energies at
// tv.py:166-169).  numpy reduces a contiguous array with its pairwise
// algorithm (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum):
//
//   PW(a, n) = n < 8    : ((0 + a0) + a1) + ...
//              n <= 128 : 8 strided accumulators r_j = a_j + a_{j+8} + ...,
//                         ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 tail
//              else     : PW(a, n2) + PW(a+n2, n-n2),  n2 = n/2 rounded down to a multiple of 8
//
// (verified bitwise against np.sum on 2-D arrays up to 2e6 elements, see
// tests/test_oracle_golden.py::test_numpy_pairwise_restatement).  Because
// the recursion splits every node above depth ds into two, the tree's top
// ds levels are a perfect binary tree over S = 2^ds "subtrees" in index order.
// The device evaluation mirrors that exactly:
//   * one 8-lane group evaluates one subtree (its <= 4 remaining recursion
//     levels and leaves, lanes = the 8 accumulators of a leaf);
//   * a CTA owns S/G consecutive subtrees and combines them with a balanced
//     shared-memory tree (pairs (2i, 2i+1) at every level);
//   * the G CTA results (G a power of two) are combined the same way.
// Every floating-point add is the one numpy performs, in the same order, so
// the sums are bit-identical to np.sum and the FGP restart / stop / fallback
// decisions and ProxInfo match the reference exactly.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace bsgd {

// Term functors are called as f(p, t).  A functor that also stores (e.g. the FGP
// momentum update) can opt into a two-stage form, `static constexpr bool
// kTwoStage = true;` with `L load(p)` (loads only) and `term(p, const L &, t)`,
// so the fast path issues the loads of several pixels before any of their
// stores: otherwise the compiler must keep every load behind the previous
// pixel's store (it cannot prove the fields do not alias) and each pixel costs
// a full memory round trip.
template <class F, class = void>
struct pw_two_stage : std::false_type {};
template <class F>
struct pw_two_stage<F, std::void_t<decltype(F::kTwoStage)>> : std::integral_constant<bool, F::kTwoStage> {};
// pixels whose loads are issued together (F::kUnroll, default 4)
template <class F, class = void>
struct pw_unroll : std::integral_constant<int, 4> {};
template <class F>
struct pw_unroll<F, std::void_t<decltype(F::kUnroll)>> : std::integral_constant<int, F::kUnroll> {};

constexpr int kPwMaxQ = 512;   // subtrees per CTA held in shared memory
constexpr int kPwMaxK = 7;     // simultaneous sums per pass (3D dual value + commit)

__host__ __device__ inline int64_t pw_split(int64_t n) {
    const int64_t n2 = n / 2;
    return n2 - (n2 % 8);
}

// subtree s at depth ds: follow the bits of s from the root
__device__ __forceinline__ void pw_subtree(int64_t N, int ds, int64_t s, int64_t &lo, int64_t &n) {
    lo = 0;
    n = N;
    for (int lev = ds - 1; lev >= 0; --lev) {
        const int64_t n2 = pw_split(n);
        if ((s >> lev) & 1) { lo += n2; n -= n2; } else { n = n2; }
    }
}

// one leaf (n <= 128) by an 8-lane group; every lane returns the sum
template <int K, class F>
__device__ __forceinline__ void pw_leaf(int64_t lo, int64_t n, F &f, unsigned gm, int j, double (&out)[K]) {
    double t[K];
    if (n < 8) {
        if (j < n) f(lo + j, t);
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = 0.0;
        for (int i = 0; i < n; ++i)
#pragma unroll
            for (int k = 0; k < K; ++k) out[k] = rn_add(out[k], __shfl_sync(gm, t[k], i, 8));
        return;
    }
    double r[K];
    f(lo + j, r);
    const int64_t full = n - (n % 8);
    for (int64_t i = 8; i < full; i += 8) {
        f(lo + i + j, t);
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = rn_add(r[k], t[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 1, 8));
        r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 2, 8));
        r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 4, 8));
    }
    const int rem = (int)(n - full);
    if (j < rem) f(lo + full + j, t);
    for (int i = 0; i < rem; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = rn_add(r[k], __shfl_sync(gm, t[k], i, 8));
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = r[k];
}

template <int K, class F, int D>
__device__ __noinline__ void pw_node(int64_t lo, int64_t n, F &f, unsigned gm, int j, double (&out)[K]) {
    if constexpr (D == 0) {
        pw_leaf<K>(lo, n, f, gm, j, out);
    } else {
        if (n <= 128) {
            pw_leaf<K>(lo, n, f, gm, j, out);
            return;
        }
        const int64_t n2 = pw_split(n);
        double a[K], b[K];
        pw_node<K, F, D - 1>(lo, n2, f, gm, j, a);
        pw_node<K, F, D - 1>(lo + n2, n - n2, f, gm, j, b);
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = rn_add(a[k], b[k]);
    }
}

// balanced in-place tree over `count` (power of two) K-vectors in shared memory;
// result in v[0..K).  All threads of the CTA must call it.
template <int K>
__device__ __forceinline__ void pw_smem_tree(double *v, int count) {
    for (int w = count; w > 1; w >>= 1) {
        const int half = w >> 1;
        double a[K];
        const int i = threadIdx.x;
        if (i < half)
#pragma unroll
            for (int k = 0; k < K; ++k) a[k] = rn_add(v[(2 * i) * K + k], v[(2 * i + 1) * K + k]);
        __syncthreads();
        if (i < half)
#pragma unroll
            for (int k = 0; k < K; ++k) v[i * K + k] = a[k];
        __syncthreads();
    }
}

// CTA part: this CTA's subtrees -> one K-vector (written to part[blockIdx.x]).
// Returns the number of subtrees this CTA owned (0 means it wrote nothing).
// Subtrees are evaluated in rounds of one per 8-lane group; each round's
// (power-of-two, aligned) run is folded by a balanced tree -- exactly the
// lower levels of the balanced tree over all Q -- so `sm` only holds one
// K-vector per round: Q <= kPwMaxQ * (blockDim.x / 8).
template <int K, class F>
__device__ __forceinline__ int pw_cta(int64_t N, int ds, F &f, double *sm, double *part) {
    __shared__ double lv[(kThreads / 8) * kPwMaxK];
    const int64_t S = (int64_t)1 << ds;
    const int G = gridDim.x;
    int64_t first;
    int Q;
    if (S >= G) {
        Q = (int)(S / G);
        first = (int64_t)blockIdx.x * Q;
    } else {
        Q = ((int64_t)blockIdx.x < S) ? 1 : 0;
        first = blockIdx.x;
    }
    const int lane = threadIdx.x & 31;
    const int j = lane & 7;
    const unsigned gm = 0xFFu << (lane & 24);
    const int group = threadIdx.x >> 3;
    const int ngroups = blockDim.x >> 3;
    int rounds = 0;
    for (int q0 = 0; q0 < Q; q0 += ngroups, ++rounds) {
        const int nq = (Q - q0 < ngroups) ? Q - q0 : ngroups;
        if (group < nq) {
            int64_t lo, n;
            pw_subtree(N, ds, first + q0 + group, lo, n);
            double v[K];
            pw_node<K, F, 4>(lo, n, f, gm, j, v);
            if (j == 0)
#pragma unroll
                for (int k = 0; k < K; ++k) lv[group * K + k] = v[k];
        }
        __syncthreads();
        pw_smem_tree<K>(lv, nq);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) sm[rounds * K + k] = lv[k];
        __syncthreads();
    }
    if (Q > 0) {
        pw_smem_tree<K>(sm, rounds);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) part[(size_t)blockIdx.x * K + k] = sm[k];
    }
    __syncthreads();
    return Q;
}

// top part: combine the min(S, G) CTA results (a power of two) in a balanced
// tree; every thread receives the totals.  `part` was written by pw_cta of a
// G-CTA grid (visible: after a grid barrier or in a later launch).  G <= 512,
// `sm` holds kPwMaxQ * K doubles.
template <int K>
__device__ __forceinline__ void pw_top(int ds, int G, const double *part, double *sm, double (&out)[K]) {
    const int64_t S = (int64_t)1 << ds;
    const int cnt = (int)(S < (int64_t)G ? S : (int64_t)G);
    for (int i = threadIdx.x; i < cnt * K; i += blockDim.x) sm[i] = __ldcg(part + i);
    __syncthreads();
    pw_smem_tree<K>(sm, cnt);
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = sm[k];
    __syncthreads();
}

// Fast path for N = 128 * 2^ds (every power-of-two image >= 16 x 16): each
// subtree is one full 128-element leaf.  Terms are produced by all threads in
// coalesced order into shared memory (CH leaves at a time), then thread
// (leaf, j) runs accumulator j's sequential chain over the leaf's 16 strided
// terms and an 8-lane butterfly forms ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)).
// Each chunk's CH leaves (an aligned power-of-two run) are folded by a
// balanced tree at once, so `leafv` holds one K-vector per chunk:
// Q <= kPwMaxQ * CH.  T holds K * CH * 128 doubles.
constexpr int kPwChunk = 16;   // default leaves per chunk

template <int K, class F, int CH = kPwChunk>
__device__ __forceinline__ int pw_cta_fast(int ds, F &f, double *T, double *leafv, double *part) {
    __shared__ double lv[kPwChunk * kPwMaxK];
    static_assert(CH <= kPwChunk && CH * 8 <= kThreads, "chunk too large");
    const int64_t S = (int64_t)1 << ds;
    const int G = gridDim.x;
    int64_t first;
    int Q;
    if (S >= G) {
        Q = (int)(S / G);
        first = (int64_t)blockIdx.x * Q;
    } else {
        Q = ((int64_t)blockIdx.x < S) ? 1 : 0;
        first = blockIdx.x;
    }
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    int chunks = 0;
    for (int c0 = 0; c0 < Q; c0 += CH, ++chunks) {
        const int nl = (Q - c0 < CH) ? Q - c0 : CH;
        const int npx = nl * 128;
        const int64_t px0 = (first + c0) * 128;
        if constexpr (pw_two_stage<F>::value) {
            constexpr int U = pw_unroll<F>::value;
            for (int i0 = tid; i0 < npx; i0 += U * (int)blockDim.x) {
                typename F::L ld[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * (int)blockDim.x;
                    if (i < npx) ld[u] = f.load(px0 + i);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + u * (int)blockDim.x;
                    if (i < npx) {
                        double t[K];
                        f.term(px0 + i, ld[u], t);
#pragma unroll
                        for (int k = 0; k < K; ++k) T[k * (CH * 128) + i] = t[k];
                    }
                }
            }
        } else {
            for (int i = tid; i < npx; i += blockDim.x) {
                double t[K];
                f(px0 + i, t);
#pragma unroll
                for (int k = 0; k < K; ++k) T[k * (CH * 128) + i] = t[k];
            }
        }
        __syncthreads();
        if (tid < nl * 8) {
            const int leaf = tid >> 3, j = tid & 7;
            const unsigned gm = 0xFFu << (lane & 24);
            double r[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double *src = T + k * (CH * 128) + leaf * 128 + j;
                double acc = src[0];
#pragma unroll
                for (int i = 1; i < 16; ++i) acc = rn_add(acc, src[8 * i]);
                r[k] = acc;
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 1, 8));
                r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 2, 8));
                r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 4, 8));
            }
            if (j == 0)
#pragma unroll
                for (int k = 0; k < K; ++k) lv[leaf * K + k] = r[k];
        }
        __syncthreads();
        pw_smem_tree<K>(lv, nl);
        if (tid == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) leafv[chunks * K + k] = lv[k];
        __syncthreads();
    }
    if (Q > 0) {
        pw_smem_tree<K>(leafv, chunks);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) part[(size_t)blockIdx.x * K + k] = leafv[k];
    }
    __syncthreads();
    return Q;
}

// Fast path without the staging buffer: thread (leaf, j) evaluates accumulator
// j's 16 strided terms of its leaf directly (8 lanes read 8 consecutive
// voxels: two full sectors per leaf per step), so a warp sums four leaves on
// its own, with no CTA barrier per chunk and no K * CH * 128 shared buffer.
// The leaf values of the CTA's Q leaves (Q <= kPwMaxQ, a power of two) are
// then folded by one balanced tree -- the same pairwise order as pw_cta_fast.
template <int K, class F>
__device__ __forceinline__ int pw_cta_direct(int ds, F &f, double *leafv, double *part) {
    const int64_t S = (int64_t)1 << ds;
    const int G = gridDim.x;
    int64_t first;
    int Q;
    if (S >= G) {
        Q = (int)(S / G);
        first = (int64_t)blockIdx.x * Q;
    } else {
        Q = ((int64_t)blockIdx.x < S) ? 1 : 0;
        first = blockIdx.x;
    }
    const int tid = threadIdx.x, lane = tid & 31;
    const int sub = lane >> 3, j = lane & 7;
    const unsigned gm = 0xFFu << (lane & 24);
    const int nw = (int)blockDim.x >> 5;
    for (int l0 = (tid >> 5) * 4; l0 < Q; l0 += nw * 4) {
        const int leaf = l0 + sub;
        double r[K];
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = 0.0;
        if (leaf < Q) {
            const int64_t base = (first + leaf) * 128 + j;
            if constexpr (pw_two_stage<F>::value) {
                constexpr int U = pw_unroll<F>::value;
                static_assert(16 % U == 0, "unroll must divide 16");
#pragma unroll 1
                for (int i0 = 0; i0 < 16; i0 += U) {
                    typename F::L ld[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) ld[u] = f.load(base + 8 * (i0 + u));
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        double t[K];
                        f.term(base + 8 * (i0 + u), ld[u], t);
#pragma unroll
                        for (int k = 0; k < K; ++k) r[k] = (i0 + u == 0) ? t[k] : rn_add(r[k], t[k]);
                    }
                }
            } else {
#pragma unroll 4
                for (int i = 0; i < 16; ++i) {
                    double t[K];
                    f(base + 8 * i, t);
#pragma unroll
                    for (int k = 0; k < K; ++k) r[k] = (i == 0) ? t[k] : rn_add(r[k], t[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 1, 8));
            r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 2, 8));
            r[k] = rn_add(r[k], __shfl_xor_sync(gm, r[k], 4, 8));
        }
        if (j == 0 && leaf < Q)
#pragma unroll
            for (int k = 0; k < K; ++k) leafv[leaf * K + k] = r[k];
    }
    __syncthreads();
    if (Q > 0) {
        pw_smem_tree<K>(leafv, Q);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < K; ++k) part[(size_t)blockIdx.x * K + k] = leafv[k];
    }
    __syncthreads();
    return Q;
}

// Balanced pairwise tree over count (a power of two) values v[i * K] in index
// order, by one warp: lane l folds its count/32 consecutive values with a
// balanced local tree, then xor butterflies combine lanes (2l, 2l+1), ...;
// the additions are commutative, so every lane ends with the bits of the
// (2i, 2i+1)-paired tree that pw_smem_tree computes.  count < 32: lanes
// >= count carry duplicates that never reach lanes < count.
// balanced tree over P consecutive values (P a power of two), fully unrolled
template <int P, class L>
__device__ __forceinline__ double fold_run(const L &ld, int base) {
    double loc[P];
#pragma unroll
    for (int i = 0; i < P; ++i) loc[i] = ld(base + i);
#pragma unroll
    for (int wdt = P; wdt > 1; wdt >>= 1)
#pragma unroll
        for (int i = 0; i < wdt / 2; ++i) loc[i] = rn_add(loc[2 * i], loc[2 * i + 1]);
    return loc[0];
}

template <int K, bool GLOBAL>
__device__ __forceinline__ double warp_pw_tree(const double *v, int count, int lane) {
    auto ld = [&](int i) { return GLOBAL ? __ldcg(v + (size_t)i * K) : v[(size_t)i * K]; };
    double acc;
    int levels = count;
    if (count >= 32) {
        const int per = count >> 5, base = lane * per;
        switch (per) {
            case 1: acc = fold_run<1>(ld, base); break;
            case 2: acc = fold_run<2>(ld, base); break;
            case 4: acc = fold_run<4>(ld, base); break;
            case 8: acc = fold_run<8>(ld, base); break;
            case 16: acc = fold_run<16>(ld, base); break;
            default: {   // 32 .. 128 per lane (count <= 4096): a balanced tree over runs of 16
                const int nc = per >> 4;
                double c[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) c[j] = j < nc ? fold_run<16>(ld, base + 16 * j) : 0.0;
#pragma unroll
                for (int wdt = 8; wdt > 1; wdt >>= 1)
                    if (wdt <= nc)
#pragma unroll
                        for (int i = 0; i < wdt / 2; ++i) c[i] = rn_add(c[2 * i], c[2 * i + 1]);
                acc = c[0];
                break;
            }
        }
        levels = 32;
    } else {
        acc = ld(lane < count ? lane : 0);
    }
    for (int off = 1; off < levels; off <<= 1) acc = rn_add(acc, __shfl_xor_sync(0xffffffffu, acc, off));
    return acc;
}

// pw_top by warps: warp k < K folds sum k of the G CTA partials (G a power of two,
// <= 512) with warp_pw_tree -- the same balanced tree as pw_top's, no CTA-wide
// barriers per level.  Every thread receives the totals.  `sm` holds K doubles.
template <int K>
__device__ __forceinline__ void pw_top_warps(int ds, int G, const double *part, double *sm, double (&out)[K]) {
    const int64_t S = (int64_t)1 << ds;
    const int cnt = (int)(S < (int64_t)G ? S : (int64_t)G);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (int)blockDim.x >> 5;
    for (int k = warp; k < K; k += nw) {
        const double v = warp_pw_tree<K, true>(part + k, cnt, lane);
        if (lane == 0) sm[k] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = sm[k];
    __syncthreads();
}

}  // namespace bsgd
