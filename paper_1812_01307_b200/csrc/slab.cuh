// Pass-per-kernel TV prox: the FGP of fgp.cuh split into one kernel per pass.
//
// Two users:
//
// 1. Multi-GPU slab decomposition (SURVEY.md §8 e, "Prox").  Rank p owns the
//    voxels [off, off + n) of the C-order volume (2-D: image) and holds every
//    field over [off - h, off + n + h), h = one plane (H*W in 3-D, W in 2-D):
//    the stencils of tv.py:115-132 (and their 3-D restatement) reach one plane
//    either way, so a one-plane halo exchanged between neighbouring ranks is all
//    a pass needs.  Field pointers are shifted so that ptr[p] addresses global
//    voxel p; boundary tests use global coordinates, so halos outside the
//    volume are never read.  The FGP decisions (restart, stop, fallback:
//    tv.py:203-253) need global sums: slabs are nodes of numpy's pairwise
//    recursion over the whole volume (parallel.prox_slabs), so a slab's local
//    numpy-order sum is exactly that node's value, and the host combines the
//    per-rank values in the recursion's order (parallel.pw_combine).  The host
//    loop (parallel.SlabProx) sequences the passes between halo exchanges.
//
// 2. Single-GPU prox of large volumes ("split" prox, launch_prox_split).  The
//    persistent cooperative fgp_kernel must keep every CTA resident and is
//    capped at 16 warps/SM by its 128-register dual pass; the candidate pass
//    alone fits in 64 registers and runs at twice the occupancy.  Here the
//    whole volume is one slab and the decisions are taken on the device by
//    one-CTA "decide" kernels into an FgpCtl block; every later pass reads the
//    block and returns at once when it does not apply (converged, or no
//    restart), so the launch sequence is fixed -- max_iters x 6 kernels -- and
//    can be captured in a CUDA graph.  Same operations in the same order as
//    fgp_kernel: bit-identical results.
#pragma once

#include "common.cuh"
#include "fgp.cuh"
#include "pairwise.cuh"

namespace bsgd {

// device-side FGP state of the split prox (fgp_kernel's registers)
struct FgpCtl {
    double phi_prev, tv_b, t_mom, t_next, beta, tv_out;
    int32_t iters, restarts, done, parity, restart, fell;
    uint32_t arrive;   // CTAs of the current sum pass that finished (folded decide)
};

struct SlabView {
    ProxArgs a;       // global D, H, W, N; b, w, step (and the split prox's outputs);
                      // f[0..DIM) dual buffer 0, f[DIM..2DIM) q, f[2DIM..3DIM) dual buffer 1,
                      // all addressed by global voxel index
    int64_t off, n;   // own voxels
    int ds;           // pairwise depth of n
    int fast;         // n == 128 * 2^ds
    int G;            // CTAs of the sum passes (entries in part)
    int parity;       // host loop: dual buffer holding p
    int when;         // split prox: 0 always, 1 unless converged, 2 only on a restart
    double *u;        // finalize output; NULL: the dual buffer not holding p
    FgpCtl *ctl;      // split prox control block, NULL for the host loop
    int zero;         // split prox, first iteration: p = q = 0 are not stored, read as zeros
    // solver vectors of step / output: 0 = full-length in volume order (vec[p]);
    // > 0 = the rank's own slices in the interleaved order of A2 (x) I_{ilv}
    // (vec[(p mod H W) * ilv + p / (H W) - z0], slice ownership of configs[4])
    int64_t ilv, ilv_z0;
    // split prox: the sum pass's last CTA to finish runs the decision of stage
    // fold_stage (iteration fold_it) itself -- no separate decide launch; -1: off
    int fold_stage, fold_it;
};

__device__ __forceinline__ int64_t slab_vec_index(const SlabView &s, int64_t p) {
    if (s.ilv == 0) return p;
    const int64_t hw = s.a.H * s.a.W;
    const int64_t z = p / hw;
    return (p - z * hw) * s.ilv + (z - s.ilv_z0);
}

__device__ __forceinline__ bool slab_skip(const SlabView &s) {
    if (s.ctl == nullptr || s.when == 0) return false;
    const FgpCtl *c = s.ctl;
    if (s.when == 1) return c->done != 0;
    return c->done != 0 || c->restart == 0;
}

template <int DIM>
struct SlabRoles {
    const double *P[DIM];
    double *C[DIM];
    double *Q[DIM];
    double *u;
};

template <int DIM>
__device__ __forceinline__ SlabRoles<DIM> slab_roles(const SlabView &s) {
    const int par = s.ctl != nullptr ? s.ctl->parity : s.parity;
    SlabRoles<DIM> r;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        r.P[k] = par ? s.a.f[2 * DIM + k] : s.a.f[k];
        r.C[k] = par ? s.a.f[k] : s.a.f[2 * DIM + k];
        r.Q[k] = s.a.f[DIM + k];
    }
    r.u = s.u != nullptr ? s.u : r.C[0];
    return r;
}

__device__ __forceinline__ void fgp_next_beta(FgpCtl &c) {
    c.t_next = 0.5 * (1.0 + sqrt(rn_add(1.0, rn_mul(rn_mul(4.0, c.t_mom), c.t_mom))));
    c.beta = (c.t_mom - 1.0) / c.t_next;
}

// stage 0: after the setup sums; 1: after the candidate's dual pass; 2: after
// the restart's dual pass; 3: after the energy sums (fallback decision, outputs).
// The same scalar code as fgp_kernel; v = the stage's global numpy-order sums.
template <int DIM>
__device__ __forceinline__ void fgp_decide(FgpCtl &c, const ProxArgs &a, int stage, int it, const double *v) {
    if (stage == 0) {
        c.phi_prev = v[0];
        c.tv_b = v[1];
        c.t_mom = 1.0;
        c.tv_out = 0.0;
        c.iters = c.restarts = c.done = c.parity = c.restart = c.fell = 0;
        fgp_next_beta(c);
        if (a.dual != nullptr) a.dual[0] = c.phi_prev;
        return;
    }
    if (stage == 3) {
        const double two_w = 2.0 * a.w;
        const double obj_out = rn_add(v[0], rn_mul(two_w, v[1]));
        const double obj_b = rn_add(0.0, rn_mul(two_w, c.tv_b));
        c.fell = obj_out > obj_b ? 1 : 0;
        c.tv_out = v[1];
        if (a.scal != nullptr) {
            a.scal[0] = c.fell ? c.tv_b : v[1];
            a.scal[1] = c.iters; a.scal[2] = c.restarts; a.scal[3] = c.done; a.scal[4] = c.fell;
        }
        if (a.info != nullptr) {
            a.info[0] = c.iters; a.info[1] = c.done; a.info[2] = c.restarts; a.info[3] = c.fell;
        }
        return;
    }
    const double phi = v[0];
    if (stage == 1 && phi > c.phi_prev) {  // restart from the last accepted point (tv.py:217-231)
        c.restart = 1;
        ++c.restarts;
        c.t_mom = 1.0;
        fgp_next_beta(c);
        return;
    }
    c.restart = 0;
    c.parity ^= 1;  // p <- c
    c.phi_prev = (c.phi_prev < phi) ? c.phi_prev : phi;
    c.t_mom = c.t_next;
    c.iters = it + 1;
    if (a.dual != nullptr) a.dual[it + 1] = c.phi_prev;
    double ch2 = rn_add(v[1], v[2]), sc2 = rn_add(v[1 + DIM], v[2 + DIM]);
    if constexpr (DIM == 3) { ch2 = rn_add(ch2, v[3]); sc2 = rn_add(sc2, v[6]); }
    const double change = sqrt(ch2), scale = sqrt(sc2);
    const double floor_scale = (1e-30 > scale) ? 1e-30 : scale;
    if (change <= a.tol * floor_scale) c.done = 1;
    else fgp_next_beta(c);
}

// The last CTA of a sum pass (all CTAs' partials visible after their fences)
// folds the CTA partials in pw_top's order and takes the stage's decision.
template <int DIM, int K>
__device__ __forceinline__ void slab_fold_decide(const SlabView &s, const double *part) {
    if (s.fold_stage < 0) return;
    __shared__ int last;
    __shared__ double sm[kPwMaxK];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&s.ctl->arrive, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double v[K];
    pw_top_warps<K>(s.ds, s.G, part, sm, v);
    if (threadIdx.x == 0) {
        fgp_decide<DIM>(*s.ctl, s.a, s.fold_stage, s.fold_it, v);
        s.ctl->arrive = 0;
    }
}

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

// The dual pass of the single-GPU split prox also writes u' = b + w div q' for the
// NEXT iteration's candidate (slab_cand_u_kernel), so no separate u pass runs
// between them: q' at the three forward neighbours is recomputed here from c
// (already loaded for div c) and p there (three extra loads, L1 / L2 hits) with
// the very operations the neighbours' own threads commit -- the same bits.
template <int DIM>
struct DualSlabTermsU : DualSlabTerms<DIM> {
    using Base = DualCommitTerms<DIM>;
    double *U;
    struct L {
        typename Base::L l;
        double pn[DIM];
    };
    __device__ __forceinline__ L load(int64_t i) const {
        L x;
        const int64_t p = this->off + i;
        x.l = Base::load(p);
        int64_t z, s, t;
        split_index<DIM>(p, this->H, this->W, z, s, t);
        const int64_t coord[3] = {z, s, t};
        const int64_t ext[3] = {this->D, this->H, this->W};
        const int64_t step[3] = {this->H * this->W, this->W, 1};
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const int ax = 3 - DIM + k;
            x.pn[k] = (this->pzero || coord[ax] + 1 >= ext[ax]) ? 0.0 : ldcg(this->P[k] + p + step[ax]);
        }
        return x;
    }
    __device__ __forceinline__ void term(int64_t i, const L &x, double (&t)[1 + 2 * DIM]) const {
        const int64_t p = this->off + i;
        Base::term(p, x.l, t);
        // div q' in div_at's order; q'_k = c_k + beta (c_k - p_k) here and at the forward neighbour
        double d = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const double qh = rn_add(x.l.here[k], rn_mul(this->beta, rn_sub(x.l.here[k], x.l.p[k])));
            const double back = (x.l.first >> k) & 1u ? 0.0 : qh;
            const double qn = rn_add(x.l.next[k], rn_mul(this->beta, rn_sub(x.l.next[k], x.pn[k])));
            d = (k == 0) ? rn_sub(qn, back) : rn_sub(rn_add(d, qn), back);
        }
        U[p] = rn_add(x.l.b, rn_mul(this->w, d));
    }
    __device__ __forceinline__ void operator()(int64_t i, double (&t)[1 + 2 * DIM]) const { term(i, load(i), t); }
};

template <int K, bool FAST, class F>
__device__ __forceinline__ void slab_sum(const SlabView &s, F &f, double *part) {
    __shared__ double sm[kPwMaxQ * kPwMaxK];
    if constexpr (FAST) pw_cta_direct<K>(s.ds, f, sm, part);   // no staging buffer, no per-chunk barriers
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
        const int64_t k = slab_vec_index(s, p);
        b[p] = rn_add(xk[k], rn_mul(mu, g[k]));
    }
}

// np.sum(b * b) and TV(b) over the own voxels (tv.py:203; tv.py:166-169 at p = 0)
// (|v - ref|^2 or |v|^2, TV(v)) per voxel as a two-stage functor (pairwise.cuh):
// the loads of kUnroll voxels (v and its three backward neighbours) are issued
// before any arithmetic -- the setup / fallback-energy sums were latency-bound
// at 1.7-2.5 TB/s as plain lambdas.  Same operations as tv_term, same bits.
template <int DIM>
struct TvSumTerms {
    static constexpr bool kTwoStage = true;
    static constexpr int kUnroll = 4;
    const double *v, *ref;   // ref NULL: t0 = v^2 (tv.py:203), else (v - ref)^2 (tv.py:166-169)
    int64_t off, H, W;
    struct L {
        double c, up, left, below;   // v at p, p - W, p - 1, p - H W (0 where absent)
        double r;
        unsigned has;                // bit 0: row > 0, bit 1: column > 0, bit 2: plane > 0
    };
    __device__ __forceinline__ L load(int64_t i) const {
        L l;
        const int64_t p = off + i;
        int64_t z, s, t;
        split_index<DIM>(p, H, W, z, s, t);
        l.has = (s > 0 ? 1u : 0u) | (t > 0 ? 2u : 0u) | (z > 0 ? 4u : 0u);
        l.c = __ldg(v + p);
        l.up = s > 0 ? __ldg(v + p - W) : 0.0;
        l.left = t > 0 ? __ldg(v + p - 1) : 0.0;
        l.below = (DIM == 3 && z > 0) ? __ldg(v + p - H * W) : 0.0;
        l.r = ref != nullptr ? __ldg(ref + p) : 0.0;
        return l;
    }
    __device__ __forceinline__ void term(int64_t, const L &l, double (&t)[2]) const {
        if (ref != nullptr) {
            const double d = rn_sub(l.c, l.r);
            t[0] = rn_mul(d, d);
        } else {
            t[0] = rn_mul(l.c, l.c);
        }
        const double dv = (l.has & 1u) ? rn_sub(l.c, l.up) : 0.0;
        const double dh = (l.has & 2u) ? rn_sub(l.c, l.left) : 0.0;
        if constexpr (DIM == 2) {
            t[1] = sqrt(rn_add(rn_mul(dv, dv), rn_mul(dh, dh)));
        } else {
            const double dz = (l.has & 4u) ? rn_sub(l.c, l.below) : 0.0;
            t[1] = sqrt(rn_add(rn_add(rn_mul(dz, dz), rn_mul(dv, dv)), rn_mul(dh, dh)));
        }
    }
    __device__ __forceinline__ void operator()(int64_t i, double (&t)[2]) const { term(i, load(i), t); }
};

template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads) slab_init_kernel(SlabView s, double *part) {
    TvSumTerms<DIM> f;
    f.v = s.a.b;
    f.ref = nullptr;
    f.off = s.off; f.H = s.a.H; f.W = s.a.W;
    slab_sum<2, FAST>(s, f, part);
    slab_fold_decide<DIM, 2>(s, part);
}

// c = proj(src + step grad(b + w div src)) on the own voxels (tv.py:207-214)
template <int DIM>
__global__ void __launch_bounds__(kThreads) slab_candidate_kernel(SlabView s, int from_p) {
    if (slab_skip(s)) return;
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    const double *src[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) src[k] = from_p ? r.P[k] : r.Q[k];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        double c[DIM];
        if (s.zero) candidate_zero<DIM>(s.a, p, c);
        else candidate<DIM>(s.a, src, p, c);
#pragma unroll
        for (int k = 0; k < DIM; ++k) r.C[k][p] = c[k];
    }
}

// The candidate from a stored u field (split prox of one GPU, where u's
// neighbours are not rewritten by another rank; u = b + w div q is written by
// the previous dual pass, slab_dual_u_kernel): c = proj(q + step grad u) from u
// and its three backward neighbours.  The fused candidate evaluates u four times
// per voxel (~590 instructions, issue-bound); the same operations in the same
// order, so c is bit-identical to slab_candidate_kernel's.
template <int DIM, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) slab_cand_u_kernel(SlabView s, int from_p, const double *u) {
    if (slab_skip(s)) return;
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    const double *src[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) src[k] = from_p ? r.P[k] : r.Q[k];
    const int64_t H = s.a.H, W = s.a.W;
    // first iteration (q = 0): u = b + w * 0 equals b except that -0 becomes +0,
    // and every gradient built from it gives the same c (0 + step * (+-0) = +0),
    // so the candidate reads b and no u pass runs
    if (s.zero) u = s.a.b;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        int64_t z, y, t;
        split_index<DIM>(p, H, W, z, y, t);
        const double uc = u[p];
        double g[DIM];
        if constexpr (DIM == 3) g[0] = (z > 0) ? rn_sub(uc, u[p - H * W]) : 0.0;
        g[DIM - 2] = (y > 0) ? rn_sub(uc, u[p - W]) : 0.0;
        g[DIM - 1] = (t > 0) ? rn_sub(uc, u[p - 1]) : 0.0;
        double c[DIM];
#pragma unroll
        for (int k = 0; k < DIM; ++k) c[k] = rn_add(s.zero ? 0.0 : src[k][p], rn_mul(s.a.step, g[k]));
        project_unit<DIM>(c);
#pragma unroll
        for (int k = 0; k < DIM; ++k) r.C[k][p] = c[k];
    }
}

// dual value of c and the speculative momentum commit q = c + beta (c - p)
// (tv.py:215-216, 233-245): 1 + 2 DIM sums.  beta from the control block when set.
// 4 CTAs per SM (60 registers, no spills): the 512 CTAs of a 256^3 pass are
// resident at once (256^3 prox 6.73 -> 6.23-6.29 ms against 2 per SM)
template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads, 4) slab_dual_u_kernel(SlabView s, double *part, double *u) {
    if (slab_skip(s)) return;
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    DualSlabTermsU<DIM> f;
    f.b = s.a.b; f.w = s.a.w;
    f.beta = s.ctl->beta;
    f.D = s.a.D; f.H = s.a.H; f.W = s.a.W;
#pragma unroll
    for (int k = 0; k < DIM; ++k) { f.P[k] = r.P[k]; f.Q[k] = r.Q[k]; f.C[k] = r.C[k]; }
    f.off = s.off;
    f.pzero = s.zero != 0;
    f.U = u;
    slab_sum<1 + 2 * DIM, FAST>(s, f, part);
    slab_fold_decide<DIM, 1 + 2 * DIM>(s, part);
}

template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads, 4) slab_dual_kernel(SlabView s, double beta, double *part) {
    if (slab_skip(s)) return;
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    DualSlabTerms<DIM> f;
    f.b = s.a.b; f.w = s.a.w;
    f.beta = s.ctl != nullptr ? s.ctl->beta : beta;
    f.D = s.a.D; f.H = s.a.H; f.W = s.a.W;
#pragma unroll
    for (int k = 0; k < DIM; ++k) { f.P[k] = r.P[k]; f.Q[k] = r.Q[k]; f.C[k] = r.C[k]; }
    f.off = s.off;
    f.pzero = s.zero != 0;
    slab_sum<1 + 2 * DIM, FAST>(s, f, part);
    slab_fold_decide<DIM, 1 + 2 * DIM>(s, part);
}

// u = b + w div p (tv.py:250)
template <int DIM>
__global__ void __launch_bounds__(kThreads) slab_finalize_kernel(SlabView s) {
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        int64_t z, y, t;
        split_index<DIM>(p, s.a.H, s.a.W, z, y, t);
        r.u[p] = rn_add(__ldg(s.a.b + p), rn_mul(s.a.w, div_at<DIM>(r.P, z, y, t, s.a.D, s.a.H, s.a.W)));
    }
}

// np.sum((u - b)^2) and TV(u) (tv.py:166-169, 251)
template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads) slab_energy_kernel(SlabView s, double *part) {
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    TvSumTerms<DIM> f;
    f.v = r.u;
    f.ref = s.a.b;
    f.off = s.off; f.H = s.a.H; f.W = s.a.W;
    slab_sum<2, FAST>(s, f, part);
    slab_fold_decide<DIM, 2>(s, part);
}

// x_next on the own voxels (identity fallback when fell) and the epoch
// statistics partials |x|^2, |x - x*|^2, d.g, |d|^2 (as fgp_kernel's epoch mode)
template <int DIM>
__global__ void __launch_bounds__(kThreads) slab_output_kernel(SlabView s, int fell, double *xn, const double *xk,
                                                               const double *g, const double *xtrue, double *part) {
    __shared__ double sm[4 * (kThreads / 32)];
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    if (s.ctl != nullptr) fell = s.ctl->fell;   // device decisions
    double st[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = s.off + i;
        const int64_t k = slab_vec_index(s, p);
        const double xv = fell ? __ldg(s.a.b + p) : __ldg(r.u + p);
        xn[k] = xv;
        const double d = rn_sub(xv, xk[k]);
        st[0] += xv * xv;
        if (xtrue != nullptr) { const double e = xv - xtrue[k]; st[1] += e * e; }
        st[2] += d * g[k];
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

// ---- split prox: device-side decisions ----

template <int DIM, int K>
__global__ void __launch_bounds__(kThreads) split_decide_kernel(SlabView s, int stage, int it, const double *part) {
    if (slab_skip(s)) return;
    __shared__ double sm[kPwMaxK];
    double v[K];
    pw_top_warps<K>(s.ds, s.G, part, sm, v);
    if (threadIdx.x != 0) return;
    fgp_decide<DIM>(*s.ctl, s.a, stage, it, v);
}

// Multi-GPU slab prox with the decisions on the device (graph-capturable): the
// ranks' slab sums, all-gathered rank-major into `gathered` (world x K), are
// combined in numpy's recursion order by a postfix program computed once on the
// host from the slab nodes (parallel.slab_program: op >= 0 pushes rank op's
// sums, -1 adds the top two), then the same decision code runs on every rank.
constexpr int kSlabRanks = 16;
constexpr int kSlabProgram = 2 * kSlabRanks;
struct SlabProgram {
    int32_t n;
    int8_t op[kSlabProgram];
};

template <int DIM, int K>
__global__ void __launch_bounds__(32) slab_decide_kernel(SlabView s, int stage, int it, const double *gathered,
                                                         SlabProgram prog) {
    if (slab_skip(s) || threadIdx.x != 0) return;
    double stk[kSlabRanks][K];
    int sp = 0;
    for (int i = 0; i < prog.n; ++i) {
        const int o = prog.op[i];
        if (o >= 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) stk[sp][k] = gathered[o * K + k];
            ++sp;
        } else {
            --sp;
#pragma unroll
            for (int k = 0; k < K; ++k) stk[sp - 1][k] = rn_add(stk[sp - 1][k], stk[sp][k]);
        }
    }
    fgp_decide<DIM>(*s.ctl, s.a, stage, it, stk[0]);
}

// outputs of the split prox: the image (standalone) or x_next in vector order
// with the epoch statistics (fgp_kernel's epoch mode)
template <int DIM>
__global__ void __launch_bounds__(kThreads) split_output_kernel(SlabView s) {
    __shared__ double sm[4 * (kThreads / 32)];
    const SlabRoles<DIM> r = slab_roles<DIM>(s);
    const ProxArgs &a = s.a;
    const int fell = s.ctl->fell;
    const int64_t N = a.N;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
    if (a.out_img != nullptr) {
        for (int64_t p = tid; p < N; p += nthr) a.out_img[p] = fell ? __ldg(a.b + p) : __ldg(r.u + p);
        return;
    }
    double st[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = tid; k < N; k += nthr) {
        const int64_t p = (a.perm != nullptr) ? a.perm[k] : k;
        const double xv = fell ? __ldg(a.b + p) : __ldg(r.u + p);
        a.x_next[k] = xv;
        const double d = rn_sub(xv, a.x_k[k]);
        st[0] += xv * xv;
        if (a.x_true != nullptr) { const double e = xv - a.x_true[k]; st[1] += e * e; }
        st[2] += d * a.g[k];
        st[3] += d * d;
    }
    block_sum<4>(st, sm);
    if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) a.xpart[(size_t)blockIdx.x * 4 + k] = st[k];
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.nx != nullptr) a.nx[0] = gridDim.x;
}

}  // namespace bsgd
