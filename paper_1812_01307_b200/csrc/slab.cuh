// Slab-decomposed TV prox for multi-GPU runs (SURVEY.md §8 e, "Prox").
//
// Rank p owns the voxels [off, off + n) of the C-order volume (2-D: image) and
// holds every field over [off - h, off + n + h), h = one plane (H*W in 3-D, W
// in 2-D): the stencils of tv.py:115-132 (and their 3-D restatement) reach one
// plane either way, so a one-plane halo exchanged between neighbouring ranks
// is all a pass needs.  Field pointers are shifted so that ptr[p] addresses
// global voxel p; boundary tests use global coordinates, so halos outside the
// volume are never read.
//
// The FGP control flow (restart, stop, fallback: tv.py:203-253) needs global
// sums.  Slabs are nodes of numpy's pairwise recursion over the whole volume
// (parallel.prox_slabs), so a slab's local numpy-order sum is exactly that
// node's value; the host gathers the per-rank values and combines them in the
// recursion's order (parallel.pw_combine): every decision is bit-identical to
// the single-GPU kernel and to the reference.  The kernels here are the FGP
// passes of fgp.cuh on a slab; the host loop (parallel.SlabProx) sequences
// them between halo exchanges.
#pragma once

#include "common.cuh"
#include "fgp.cuh"
#include "pairwise.cuh"

namespace bsgd {

struct SlabView {
    ProxArgs a;       // global D, H, W, N; b and f[] shifted to global indexing; w, step
    int64_t off, n;   // own voxels
    int ds;           // pairwise depth of n
    int fast;         // n == 128 * 2^ds
    double *u;        // finalize output (shifted)
};

// DualCommitTerms over the slab: local index i -> voxel off + i
template <int DIM>
struct DualSlabTerms : DualCommitTerms<DIM> {
    using Base = DualCommitTerms<DIM>;
    using L = typename Base::L;
    int64_t off;
    __device__ __forceinline__ L load(int64_t i) const { return Base::load(off + i); }
    __device__ __forceinline__ void term(int64_t i, const L &l, double (&t)[1 + 2 * DIM]) const {
        Base::term(off + i, l, t);
    }
    __device__ __forceinline__ void operator()(int64_t i, double (&t)[1 + 2 * DIM]) const {
        Base::term(off + i, Base::load(off + i), t);
    }
};

template <int K, bool FAST, class F>
__device__ __forceinline__ void slab_sum(const SlabView &s, F &f, double *part) {
    __shared__ double sm[kPwMaxQ * kPwMaxK];
    extern __shared__ double Tsm[];
    if constexpr (FAST) pw_cta_fast<K, F, 8>(s.ds, f, Tsm, sm, part);
    else pw_cta<K>(s.n, s.ds, f, sm, part);
}

template <int K>
__global__ void __launch_bounds__(kThreads) slab_top_kernel(int ds, int G, const double *part, double *out) {
    __shared__ double sm[kPwMaxQ * kPwMaxK];
    double v[K];
    pw_top<K>(ds, G, part, sm, v);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = v[k];
}

// b = x_k + mu g on the own voxels (identity layout: vector order = volume order)
__global__ void __launch_bounds__(kThreads) slab_step_kernel(SlabView s, const double *xk, const double *g, double mu) {
    double *b = const_cast<double *>(s.a.b);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        b[p] = rn_add(xk[p], rn_mul(mu, g[p]));
    }
}

// np.sum(b * b) and TV(b) over the own voxels (tv.py:203; tv.py:166-169 at p = 0)
template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads) slab_init_kernel(SlabView s, double *part) {
    const double *b = s.a.b;
    const int64_t H = s.a.H, W = s.a.W, off = s.off;
    auto f = [&](int64_t i, double (&t)[2]) {
        const int64_t p = off + i;
        const double bb = __ldg(b + p);
        t[0] = rn_mul(bb, bb);
        t[1] = tv_term<DIM>(b, p, H, W, false);
    };
    slab_sum<2, FAST>(s, f, part);
}

// c = proj(src + step grad(b + w div src)) on the own voxels (tv.py:207-214)
template <int DIM>
__global__ void __launch_bounds__(kThreads) slab_candidate_kernel(SlabView s, int from_p) {
    const double *src[DIM];
    double *C[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        src[k] = from_p ? s.a.f[k] : s.a.f[DIM + k];
        C[k] = s.a.f[2 * DIM + k];
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        double c[DIM];
        candidate<DIM>(s.a, src, p, c);
#pragma unroll
        for (int k = 0; k < DIM; ++k) C[k][p] = c[k];
    }
}

// dual value of c and the speculative momentum commit q = c + beta (c - p)
// (tv.py:215-216, 233-245): 1 + 2 DIM sums
template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads, 2) slab_dual_kernel(SlabView s, double beta, double *part) {
    DualSlabTerms<DIM> f;
    f.b = s.a.b; f.w = s.a.w; f.beta = beta;
    f.D = s.a.D; f.H = s.a.H; f.W = s.a.W;
#pragma unroll
    for (int k = 0; k < DIM; ++k) { f.P[k] = s.a.f[k]; f.Q[k] = s.a.f[DIM + k]; f.C[k] = s.a.f[2 * DIM + k]; }
    f.off = s.off;
    slab_sum<1 + 2 * DIM, FAST>(s, f, part);
}

// u = b + w div p (tv.py:250)
template <int DIM>
__global__ void __launch_bounds__(kThreads) slab_finalize_kernel(SlabView s) {
    const double *P[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) P[k] = s.a.f[k];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        int64_t z, r, t;
        split_index<DIM>(p, s.a.H, s.a.W, z, r, t);
        s.u[p] = rn_add(__ldg(s.a.b + p), rn_mul(s.a.w, div_at<DIM>(P, z, r, t, s.a.D, s.a.H, s.a.W)));
    }
}

// np.sum((u - b)^2) and TV(u) (tv.py:166-169, 251)
template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads) slab_energy_kernel(SlabView s, double *part) {
    const double *b = s.a.b, *u = s.u;
    const int64_t H = s.a.H, W = s.a.W, off = s.off;
    auto f = [&](int64_t i, double (&t)[2]) {
        const int64_t p = off + i;
        const double d = rn_sub(__ldg(u + p), __ldg(b + p));
        t[0] = rn_mul(d, d);
        t[1] = tv_term<DIM>(u, p, H, W, false);
    };
    slab_sum<2, FAST>(s, f, part);
}

// x_next on the own voxels (identity fallback when fell) and the epoch
// statistics partials |x|^2, |x - x*|^2, d.g, |d|^2 (as fgp_kernel's epoch mode)
__global__ void __launch_bounds__(kThreads) slab_output_kernel(SlabView s, int fell, double *xn, const double *xk,
                                                               const double *g, const double *xtrue, double *part) {
    __shared__ double sm[4 * (kThreads / 32)];
    double st[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        const double xv = fell ? __ldg(s.a.b + p) : __ldg(s.u + p);
        xn[p] = xv;
        const double d = rn_sub(xv, xk[p]);
        st[0] += xv * xv;
        if (xtrue != nullptr) { const double e = xv - xtrue[p]; st[1] += e * e; }
        st[2] += d * g[p];
        st[3] += d * d;
    }
    block_sum<4>(st, sm);
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) part[(size_t)blockIdx.x * 4 + k] = st[k];
}

__global__ void slab_sum4_kernel(const double *part, int n, double *out) {
    double v[4];
    warp_sum_partials<4>(part, n, v);
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) out[k] = v[k];
}

}  // namespace bsgd
