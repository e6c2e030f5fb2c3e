// TV proximal step: restarted dual fast gradient projection (tv.py:172-255)
// as ONE persistent cooperative kernel per prox call.
//
// The FGP control flow is global: every inner iteration needs the dual value
// phi over the whole image before it may commit (restart test, tv.py:217),
// and the stop test needs ||c - p|| and ||c|| (tv.py:239-248).  Instead of
// ~4 launches per iteration plus host round trips, one co-resident grid
// loops over the iterations and meets at grid barriers:
//
//   A  c = proj(q + step * grad(b + w div q))          (stencil, writes c)
//   B  phi = sum (b + w div c)^2                         (stencil, grid sum)
//      phi > phi_prev -> A', B' from p (restart)         (uniform decision)
//   C  q = c + beta (c - p); ||c - p||^2, ||c||^2        (grid sum); p <- c by
//      swapping the p / c buffer pair (no copy)
//
// All decisions are taken redundantly by every CTA from the same fixed-order
// sums, so they agree without another barrier.  Fields that are rewritten
// inside the kernel are read with ld.global.cg (L2) because L1 is not
// coherent across SMs.  Elementwise arithmetic uses explicit round-to-nearest
// intrinsics (no FMA contraction) in the reference's operation order, so the
// only deviation from numpy is the order of the three global sums.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "pairwise.cuh"
#include "prox_args.cuh"

namespace bsgd {

namespace cg = cooperative_groups;


// Fields rewritten inside the kernel are only read in phases separated from
// their writes by grid.sync(), which issues MEMBAR.GPU + CCTL.IVALL (checked in
// the SASS), so plain L1-cached loads are coherent here.
__device__ __forceinline__ double ldcg(const double *p) { return *p; }

// ---- stencils, dimension-generic (DIM = 2: tv.py:115-132; DIM = 3: oracle divergence3) ----
// fields are passed as DIM pointers ordered (z,) row, column.

// div p at voxel o = ((z*H + s)*W + t):
//   2D  ((pv[s+1] - pv[s]) + ph[t+1]) - ph[t]
//   3D  ((((pz[z+1] - pz[z]) + pv[s+1]) - pv[s]) + ph[t+1]) - ph[t]      zero outside
template <int DIM>
__device__ __forceinline__ double div_at(const double *const *pf, int64_t z, int64_t s, int64_t t, int64_t D,
                                         int64_t H, int64_t W) {
    const int64_t o = (z * H + s) * W + t;
    const double *pv = pf[DIM - 2], *ph = pf[DIM - 1];
    const double a = (s + 1 < H) ? ldcg(pv + o + W) : 0.0;
    const double b = (s > 0) ? ldcg(pv + o) : 0.0;
    const double c = (t + 1 < W) ? ldcg(ph + o + 1) : 0.0;
    const double d = (t > 0) ? ldcg(ph + o) : 0.0;
    if constexpr (DIM == 2) {
        return rn_sub(rn_add(rn_sub(a, b), c), d);
    } else {
        const double *pz = pf[0];
        const double az = (z + 1 < D) ? ldcg(pz + o + H * W) : 0.0;
        const double bz = (z > 0) ? ldcg(pz + o) : 0.0;
        return rn_sub(rn_add(rn_sub(rn_add(rn_sub(az, bz), a), b), c), d);
    }
}

// voxel index -> (z, row, column); 2D skips the plane division
// (images and volumes have < 2^31 voxels, checked at the ABI: 32-bit divisions)
template <int DIM>
__device__ __forceinline__ void split_index(int64_t p, int64_t H, int64_t W, int64_t &z, int64_t &s, int64_t &t) {
    const uint32_t pp = (uint32_t)p, w = (uint32_t)W;
    uint32_t r = pp;
    z = 0;
    // power-of-two planes and rows (every configuration): shifts and masks instead
    // of two 32-bit divisions by runtime values (~20 instructions each)
    const uint32_t hw = (uint32_t)(H * W);
    if ((w & (w - 1)) == 0 && (DIM == 2 || (hw & (hw - 1)) == 0)) {
        if constexpr (DIM == 3) {
            z = pp >> (__ffs(hw) - 1);
            r = pp & (hw - 1);
        }
        s = r >> (__ffs(w) - 1);
        t = r & (w - 1);
        return;
    }
    if constexpr (DIM == 3) {
        const uint32_t hw = (uint32_t)(H * W);
        const uint32_t zz = pp / hw;
        z = zz;
        r = pp - zz * hw;
    }
    const uint32_t ss = r / w;
    s = ss;
    t = r - ss * w;
}

// legacy 2D signature (discrete_divergence kernel)
__device__ __forceinline__ double div_at(const double *pv, const double *ph, int64_t s, int64_t t, int64_t H,
                                         int64_t W) {
    const double *pf[2] = {pv, ph};
    return div_at<2>(pf, 0, s, t, 1, H, W);
}

// u = b + w div q at voxel (z, s, t)
template <int DIM>
__device__ __forceinline__ double u_at(const ProxArgs &a, const double *const *qf, int64_t z, int64_t s, int64_t t) {
    return rn_add(__ldg(a.b + (z * a.H + s) * a.W + t), rn_mul(a.w, div_at<DIM>(qf, z, s, t, a.D, a.H, a.W)));
}

// c / max(|c|, 1) (tv.py:211-214)
// Inside the unit ball (m2 < 1) sqrt(m2) <= 1, so the divisor is exactly 1.0 and
// c / 1.0 == c bit for bit: the sqrt and the divisions run only where the
// projection is active (NaN takes the division path, as np.maximum propagates it).
template <int DIM>
__device__ __forceinline__ void project_unit(double (&c)[DIM]) {
    double m2 = rn_add(rn_mul(c[0], c[0]), rn_mul(c[1], c[1]));
    if constexpr (DIM == 3) m2 = rn_add(m2, rn_mul(c[2], c[2]));
    if (!(m2 < 1.0)) {
        double mag = sqrt(m2);
        mag = (mag < 1.0) ? 1.0 : mag;  // np.maximum(mag, 1): NaN propagates
#pragma unroll
        for (int k = 0; k < DIM; ++k) c[k] = c[k] / mag;
    }
}

// projected gradient candidate from q at voxel p (tv.py:207-214; 3D: same with three fields)
template <int DIM>
__device__ __forceinline__ void candidate(const ProxArgs &a, const double *const *qf, int64_t p, double (&c)[DIM]) {
    int64_t z, s, t;
    split_index<DIM>(p, a.H, a.W, z, s, t);
    const double uc = u_at<DIM>(a, qf, z, s, t);
    double g[DIM];
    if constexpr (DIM == 3) g[0] = (z > 0) ? rn_sub(uc, u_at<DIM>(a, qf, z - 1, s, t)) : 0.0;
    g[DIM - 2] = (s > 0) ? rn_sub(uc, u_at<DIM>(a, qf, z, s - 1, t)) : 0.0;
    g[DIM - 1] = (t > 0) ? rn_sub(uc, u_at<DIM>(a, qf, z, s, t - 1)) : 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) c[k] = rn_add(ldcg(qf[k] + p), rn_mul(a.step, g[k]));
    project_unit<DIM>(c);
}

// the same candidate for q = 0 (the first FGP iteration, tv.py:198-201): every
// operation of `candidate` on literal zeros instead of loads -- div 0 is +0, so
// u = b + w * (+0) and c = (+0) + step g -- bit-identical without the zeroed fields
template <int DIM>
__device__ __forceinline__ void candidate_zero(const ProxArgs &a, int64_t p, double (&c)[DIM]) {
    int64_t z, s, t;
    split_index<DIM>(p, a.H, a.W, z, s, t);
    const double wz = rn_mul(a.w, 0.0);
    const double uc = rn_add(__ldg(a.b + p), wz);
    double g[DIM];
    if constexpr (DIM == 3) g[0] = (z > 0) ? rn_sub(uc, rn_add(__ldg(a.b + p - a.H * a.W), wz)) : 0.0;
    g[DIM - 2] = (s > 0) ? rn_sub(uc, rn_add(__ldg(a.b + p - a.W), wz)) : 0.0;
    g[DIM - 1] = (t > 0) ? rn_sub(uc, rn_add(__ldg(a.b + p - 1), wz)) : 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) c[k] = rn_add(0.0, rn_mul(a.step, g[k]));
    project_unit<DIM>(c);
}

// isotropic TV term at voxel p of u (tv.py:149-152; 3D: sqrt((dz^2 + dv^2) + dh^2))
template <int DIM>
__device__ __forceinline__ double tv_term(const double *u, int64_t p, int64_t H, int64_t W, bool cg_load) {
    const int64_t HW = H * W;
    int64_t z, s, t;
    split_index<DIM>(p, H, W, z, s, t);
    const double uc = cg_load ? ldcg(u + p) : __ldg(u + p);
    double dv = 0.0, dh = 0.0;
    if (s > 0) dv = rn_sub(uc, cg_load ? ldcg(u + p - W) : __ldg(u + p - W));
    if (t > 0) dh = rn_sub(uc, cg_load ? ldcg(u + p - 1) : __ldg(u + p - 1));
    if constexpr (DIM == 2) {
        return sqrt(rn_add(rn_mul(dv, dv), rn_mul(dh, dh)));
    } else {
        double dz = 0.0;
        if (z > 0) dz = rn_sub(uc, cg_load ? ldcg(u + p - HW) : __ldg(u + p - HW));
        return sqrt(rn_add(rn_add(rn_mul(dz, dz), rn_mul(dv, dv)), rn_mul(dh, dh)));
    }
}

// legacy 2D signature
__device__ __forceinline__ double tv_term(const double *u, int64_t p, int64_t W, bool cg_load) {
    const int64_t s = p / W;
    return tv_term<2>(u, p, s + 1, W, cg_load);
}

// numpy-order grid sum of K per-pixel terms (pairwise.cuh); all threads get the
// totals.  Term functors may write outputs: each pixel is visited once.
// leaves per term chunk of the fast path (8: keeps 2 CTAs per SM with 7 sums)
template <int DIM>
__host__ __device__ constexpr int fgp_chunk() { return 8; }

// FAST is a template parameter so that the fast-path kernel never passes the
// term functors to the out-of-line pw_node: functors that escape to a call keep
// their captured field pointers in local memory (LDL in the hot loops).
template <int K, int CH, bool FAST, class F>
__device__ __forceinline__ void np_sum(cg::grid_group &grid, int64_t N, int ds, F &f, double *red, int &round,
                                       double *sm, double (&out)[K], double *T) {
    double *buf = red + (size_t)(round & 1) * kMaxPartials * kPwMaxK;
    if constexpr (FAST) {
        // direct leaf sums when every warp has at least two 4-leaf groups and the
        // leaves fit one shared K-vector each (2048^2: 4.54 -> 2.93 ms for 20
        // iterations); staged chunks otherwise (512^2: 8 leaves per CTA would
        // leave 6 of 8 warps idle)
        const int64_t q = ((int64_t)1 << ds) / gridDim.x;
        if (q >= 64 && q <= kPwMaxQ) pw_cta_direct<K>(ds, f, sm, buf);
        else pw_cta_fast<K, F, CH>(ds, f, T, sm, buf);
    } else {
        pw_cta<K>(N, ds, f, sm, buf);
    }
    grid.sync();
    pw_top<K>(ds, gridDim.x, buf, sm, out);
    ++round;
}

// One pass for the dual value of the candidate and the momentum commit
// (tv.py:215-216 and 233-245), two-stage (pairwise.cuh):
//   t[0]           = (b + w div c)^2                        -> phi
//   t[1 .. DIM]    = (c_k - p_k)^2                         -> change
//   t[DIM+1 .. 2D] = c_k^2                                 -> scale
//   q_k            = c_k + beta (c_k - p_k)
// The commit is speculative: when phi triggers a restart the kernel recomputes
// the candidate and runs this pass again, overwriting q (same values and sums
// as the reference's restart-then-commit order).
template <int DIM>
struct DualCommitTerms {
    static constexpr bool kTwoStage = true;
    static constexpr int kUnroll = DIM == 3 ? 1 : 2;  // 3D: 10 loads per pixel already, registers are the limit
    const double *b;
    const double *C[DIM];
    const double *P[DIM];
    double *Q[DIM];
    double w, beta;
    int64_t D, H, W;
    bool pzero = false;   // p = 0 (first FGP iteration): literal zeros instead of loads
    struct L {
        double b, here[DIM], next[DIM], p[DIM];
        unsigned first;  // bit k: coordinate k is 0 (no backward neighbour)
    };
    __device__ __forceinline__ L load(int64_t p) const {
        L l;
        int64_t z, s, t;
        split_index<DIM>(p, H, W, z, s, t);
        const int64_t coord[3] = {z, s, t};
        const int64_t ext[3] = {D, H, W};
        const int64_t step[3] = {H * W, W, 1};
        l.b = __ldg(b + p);
        l.first = 0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const int ax = 3 - DIM + k;  // 2D: rows, columns; 3D: z, rows, columns
            l.here[k] = ldcg(C[k] + p);
            l.next[k] = (coord[ax] + 1 < ext[ax]) ? ldcg(C[k] + p + step[ax]) : 0.0;
            l.p[k] = pzero ? 0.0 : ldcg(P[k] + p);
            if (coord[ax] == 0) l.first |= 1u << k;
        }
        return l;
    }
    __device__ __forceinline__ void term(int64_t p, const L &l, double (&t)[1 + 2 * DIM]) const {
        // div c, in div_at's order: ((((az - bz) + av) - bv) + ah) - bh
        double d = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const double back = (l.first >> k) & 1u ? 0.0 : l.here[k];
            d = (k == 0) ? rn_sub(l.next[k], back) : rn_sub(rn_add(d, l.next[k]), back);
        }
        const double res = rn_add(l.b, rn_mul(w, d));
        t[0] = rn_mul(res, res);
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const double sk = rn_sub(l.here[k], l.p[k]);
            Q[k][p] = rn_add(l.here[k], rn_mul(beta, sk));
            t[1 + k] = rn_mul(sk, sk);
            t[1 + DIM + k] = rn_mul(l.here[k], l.here[k]);
        }
    }
    __device__ __forceinline__ void operator()(int64_t p, double (&t)[1 + 2 * DIM]) const { term(p, load(p), t); }
};

template <int DIM, bool FAST>
__global__ void __launch_bounds__(kThreads, 2) fgp_kernel(ProxArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double sm[kPwMaxQ * kPwMaxK];
    extern __shared__ double Tsm[];   // 2*DIM * CH * 128 doubles (fast path)
    constexpr int CH = fgp_chunk<DIM>();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t N = a.N, W = a.W, H = a.H, D = a.D;
    const double w = a.w;
    const double *b = a.b;
    int round = 0;
    double *P[DIM], *Q[DIM], *C[DIM];
#pragma unroll
    for (int k = 0; k < DIM; ++k) { P[k] = a.f[k]; Q[k] = a.f[DIM + k]; C[k] = a.f[2 * DIM + k]; }

    // --- setup: p = q = 0 (tv.py:198-201), phi_prev = np.sum(b*b) (tv.py:203),
    //     and TV(b) for the fallback test (tv.py:166-169, 251)
    double v2[2];
    {
        for (int64_t p = tid; p < N; p += nthr)
#pragma unroll
            for (int k = 0; k < DIM; ++k) { P[k][p] = 0.0; Q[k][p] = 0.0; }
        auto f0 = [&](int64_t p, double (&t)[2]) {
            const double bb = __ldg(b + p);
            t[0] = rn_mul(bb, bb);
            t[1] = tv_term<DIM>(b, p, H, W, false);
        };
        np_sum<2, CH, FAST>(grid, N, a.ds, f0, a.red, round, sm, v2, Tsm);
    }
    double phi_prev = v2[0];
    const double tv_b = v2[1];
    double t_mom = 1.0;
    int iters = 0, restarts = 0, converged = 0;
    if (tid == 0 && a.dual != nullptr) a.dual[0] = phi_prev;

    // c = proj(src + step grad(b + w div src)) into C, then a grid barrier; two
    // pixels per pass, both candidates before either store (see pw_two_stage).
    // (A two-pass form through a stored u = b + w div src field -- 14 loads per
    // voxel instead of 28 -- measured slower on 256^3: 15.1 vs 14.0 ms.)
    auto candidate_pass = [&](double *const *src) {
        for (int64_t p0 = tid; p0 < N; p0 += 2 * nthr) {
            const int64_t p1 = p0 + nthr;
            double c0[DIM], c1[DIM];
            candidate<DIM>(a, src, p0, c0);
            if (p1 < N) candidate<DIM>(a, src, p1, c1);
#pragma unroll
            for (int k = 0; k < DIM; ++k) C[k][p0] = c0[k];
            if (p1 < N)
#pragma unroll
                for (int k = 0; k < DIM; ++k) C[k][p1] = c1[k];
        }
        grid.sync();
    };
    DualCommitTerms<DIM> fdc;
    fdc.b = b; fdc.w = w; fdc.D = D; fdc.H = H; fdc.W = W;
    for (int it = 0; it < a.max_iters; ++it) {
        // A: candidate from q (tv.py:207-214)
        candidate_pass(Q);
        // B+C: phi = np.sum(resid * resid) (tv.py:215-216) and the momentum commit
        //    (tv.py:233-245) in one pass, the commit speculative on "no restart"
        double t_next = 0.5 * (1.0 + sqrt(rn_add(1.0, rn_mul(rn_mul(4.0, t_mom), t_mom))));
        double beta = (t_mom - 1.0) / t_next;
#pragma unroll
        for (int k = 0; k < DIM; ++k) { fdc.C[k] = C[k]; fdc.P[k] = P[k]; fdc.Q[k] = Q[k]; }
        fdc.beta = beta;
        double vc[1 + 2 * DIM];
        np_sum<1 + 2 * DIM, CH, FAST>(grid, N, a.ds, fdc, a.red, round, sm, vc, Tsm);
        double phi = vc[0];
        if (phi > phi_prev) {  // restart from the last accepted point (tv.py:217-231)
            ++restarts;
            t_mom = 1.0;
            candidate_pass(P);
            t_next = 0.5 * (1.0 + sqrt(rn_add(1.0, rn_mul(rn_mul(4.0, t_mom), t_mom))));
            beta = (t_mom - 1.0) / t_next;
            fdc.beta = beta;
            np_sum<1 + 2 * DIM, CH, FAST>(grid, N, a.ds, fdc, a.red, round, sm, vc, Tsm);
            phi = vc[0];
        }
#pragma unroll
        for (int k = 0; k < DIM; ++k) { double *tmp_ = P[k]; P[k] = C[k]; C[k] = tmp_; }  // p <- c
        phi_prev = (phi_prev < phi) ? phi_prev : phi;  // Python min(phi, phi_prev)
        t_mom = t_next;
        iters = it + 1;
        if (tid == 0 && a.dual != nullptr) a.dual[it + 1] = phi_prev;
        double ch2 = rn_add(vc[1], vc[2]), sc2 = rn_add(vc[1 + DIM], vc[2 + DIM]);
        if constexpr (DIM == 3) { ch2 = rn_add(ch2, vc[3]); sc2 = rn_add(sc2, vc[6]); }
        const double change = sqrt(ch2), scale = sqrt(sc2);
        const double floor_scale = (1e-30 > scale) ? 1e-30 : scale;  // Python max(scale, 1e-30)
        if (change <= a.tol * floor_scale) { converged = 1; break; }
    }

    // --- finalize: out = b + w div p (tv.py:250), identity fallback if the primal
    //     objective is worse (tv.py:251-253)
    double *tmp = C[0];  // scratch after the swap
    for (int64_t p0 = tid; p0 < N; p0 += 2 * nthr) {
        const int64_t p1 = p0 + nthr;
        int64_t z, s, t;
        split_index<DIM>(p0, H, W, z, s, t);
        const double v0 = rn_add(__ldg(b + p0), rn_mul(w, div_at<DIM>(P, z, s, t, D, H, W)));
        double v1 = 0.0;
        if (p1 < N) {
            split_index<DIM>(p1, H, W, z, s, t);
            v1 = rn_add(__ldg(b + p1), rn_mul(w, div_at<DIM>(P, z, s, t, D, H, W)));
        }
        tmp[p0] = v0;
        if (p1 < N) tmp[p1] = v1;
    }
    grid.sync();
    auto fen = [&](int64_t p, double (&t)[2]) {
        const double d = rn_sub(ldcg(tmp + p), __ldg(b + p));
        t[0] = rn_mul(d, d);
        t[1] = tv_term<DIM>(tmp, p, H, W, true);
    };
    double e2[2];
    np_sum<2, CH, FAST>(grid, N, a.ds, fen, a.red, round, sm, e2, Tsm);
    const double two_w = 2.0 * w;
    const double obj_out = rn_add(e2[0], rn_mul(two_w, e2[1]));
    const double obj_b = rn_add(0.0, rn_mul(two_w, tv_b));
    const int fell = obj_out > obj_b ? 1 : 0;

    if (a.out_img != nullptr) {
        for (int64_t p = tid; p < N; p += nthr) a.out_img[p] = fell ? __ldg(b + p) : ldcg(tmp + p);
    } else {
        double st[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t k = tid; k < N; k += nthr) {
            const int64_t p = (a.perm != nullptr) ? a.perm[k] : k;
            const double xv = fell ? __ldg(b + p) : ldcg(tmp + p);
            a.x_next[k] = xv;
            const double d = rn_sub(xv, a.x_k[k]);
            st[0] += xv * xv;
            if (a.x_true != nullptr) {
                const double e = xv - a.x_true[k];
                st[1] += e * e;
            }
            st[2] += d * a.g[k];
            st[3] += d * d;
        }
        block_sum<4>(st, sm);
        if (threadIdx.x == 0)
            for (int k = 0; k < 4; ++k) a.xpart[(size_t)blockIdx.x * 4 + k] = st[k];
    }
    if (tid == 0) {
        if (a.scal != nullptr) {
            a.scal[0] = fell ? tv_b : e2[1];
            a.scal[1] = iters; a.scal[2] = restarts; a.scal[3] = converged; a.scal[4] = fell;
        }
        if (a.nx != nullptr) a.nx[0] = gridDim.x;
        if (a.info != nullptr) {
            a.info[0] = iters; a.info[1] = converged; a.info[2] = restarts; a.info[3] = fell;
        }
    }
}

// elementwise step for the retry path (solvers.py:307-314 with the stored g):
// x = x_k + mu g, scattered to image order for the prox or stored with stats.
__global__ void __launch_bounds__(kThreads) step_kernel(int64_t n, const double *xk, const double *g, double mu,
                                                        double *xn, double *uimg, const int64_t *perm,
                                                        const double *xtrue, double *xpart, int64_t *nx) {
    __shared__ double sm[4 * (kThreads / 32)];
    double st[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double gg = g[k];
        const double xo = xk[k];
        const double xv = rn_add(xo, rn_mul(mu, gg));
        if (uimg != nullptr) {
            uimg[perm != nullptr ? perm[k] : k] = xv;
        } else {
            xn[k] = xv;
            const double d = rn_sub(xv, xo);
            st[0] += xv * xv;
            if (xtrue != nullptr) { const double e = xv - xtrue[k]; st[1] += e * e; }
            st[2] += d * gg;
            st[3] += d * d;
        }
    }
    if (uimg == nullptr) {
        block_sum<4>(st, sm);
        if (threadIdx.x == 0)
            for (int k = 0; k < 4; ++k) xpart[(size_t)blockIdx.x * 4 + k] = st[k];
        if (blockIdx.x == 0 && threadIdx.x == 0) nx[0] = gridDim.x;
    }
}

// ---- small image kernels (tv.py:115-152) ----
// tv_value in numpy order: CTA part (grid of G = power of two CTAs) ...
template <int DIM>
__global__ void __launch_bounds__(kThreads) tv_value_part_kernel(int64_t D, int64_t H, int64_t W, const double *u,
                                                                 int ds, double *part) {
    __shared__ double sm[kPwMaxQ];
    auto f = [&](int64_t p, double (&t)[1]) { t[0] = tv_term<DIM>(u, p, H, W, false); };
    pw_cta<1>(D * H * W, ds, f, sm, part);
}
// ... and the balanced top over the CTA parts (one CTA)
__global__ void __launch_bounds__(kThreads) pw_top_kernel(int ds, int G, const double *part, double *out) {
    __shared__ double sm[kPwMaxQ];
    double v[1];
    pw_top<1>(ds, G, part, sm, v);
    if (threadIdx.x == 0) out[0] = v[0];
}

__global__ void __launch_bounds__(kThreads) gradient3_kernel(int64_t D, int64_t H, int64_t W, const double *u,
                                                             double *dz, double *dv, double *dh) {
    const int64_t HW = H * W;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < D * HW; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = p / HW, r = p - z * HW, s = r / W, t = r - s * W;
        dz[p] = z > 0 ? rn_sub(u[p], u[p - HW]) : 0.0;
        dv[p] = s > 0 ? rn_sub(u[p], u[p - W]) : 0.0;
        dh[p] = t > 0 ? rn_sub(u[p], u[p - 1]) : 0.0;
    }
}

__global__ void __launch_bounds__(kThreads) divergence3_kernel(int64_t D, int64_t H, int64_t W, const double *pz,
                                                               const double *pv, const double *ph, double *out) {
    const int64_t HW = H * W;
    const double *pf[3] = {pz, pv, ph};
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < D * HW; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = p / HW, r = p - z * HW, s = r / W, t = r - s * W;
        out[p] = div_at<3>(pf, z, s, t, D, H, W);
    }
}

__global__ void __launch_bounds__(kThreads) gradient_kernel(int64_t H, int64_t W, const double *u, double *dv,
                                                            double *dh) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < H * W; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = p / W, t = p - s * W;
        dv[p] = s > 0 ? rn_sub(u[p], u[p - W]) : 0.0;
        dh[p] = t > 0 ? rn_sub(u[p], u[p - 1]) : 0.0;
    }
}

__global__ void __launch_bounds__(kThreads) divergence_kernel(int64_t H, int64_t W, const double *pv,
                                                              const double *ph, double *out) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < H * W; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = p / W, t = p - s * W;
        out[p] = div_at(pv, ph, s, t, H, W);
    }
}

}  // namespace bsgd
