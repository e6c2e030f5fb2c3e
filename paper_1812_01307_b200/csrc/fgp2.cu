// 2-D TV prox (tv.py:172-255) as a row-walk persistent kernel: ONE grid
// barrier per FGP iteration instead of two, stencils from registers instead of
// re-derived neighbour loads.
//
// Geometry: G = 128 (or fewer, a power of two) co-resident CTAs; CTA g owns
// the R = H / G consecutive rows [r0, r1) -- N / G consecutive pixels, i.e. a
// complete subtree of numpy's pairwise tree (pairwise.cuh), so the CTA results
// combine exactly as np.sum does.  Thread tau owns columns 2 tau, 2 tau + 1
// (W / 2 threads, 16-byte loads) and walks down the CTA's rows.
//
// One pass per FGP iteration fuses the candidate (tv.py:207-214) and the dual
// value + momentum commit (tv.py:215-216, 233-245) as a three-stage software
// pipeline over rows, stage X at step k handling row r0 - d_X + k:
//
//   U  u(s) = b + w div q (s)                    loads q(s+1) / q(s) / b(s)
//   C  c(s) = proj(q(s) + step grad u(s))        u(s), u(s-1) from registers
//   B  phi, |c-p|^2, |c|^2 terms of row s,       c(s+1), c(s) from registers
//      q'(s) = c + beta (c - p), store c(s)
//
// The row below the slab (r1) is computed redundantly by the C stage, so the
// dual value needs no neighbour data that is written in the same pass: the
// only cross-CTA exchange is the q / p halo written in the PREVIOUS pass,
// visible after its grid barrier.  q is double-buffered (read Q, write Q')
// because a neighbour may still read q's halo rows while this CTA commits.
// Within a warp, column neighbours come from shuffles; across warps, through
// a per-step shared-memory exchange of the edge lanes' u and ch.  Each row's
// terms are staged in shared memory and summed by 8-lane groups in numpy's
// leaf order (8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))).
//
// Arithmetic: every elementwise operation is the reference's, in its order,
// with explicit round-to-nearest intrinsics (no FMA), and every global sum is
// numpy's pairwise sum -- the result, ProxInfo and the dual objectives are
// bit-identical to tv.py and to fgp_kernel<2> (which serves the shapes this
// kernel does not: non-power-of-two images, W > 1024).

#include <cooperative_groups.h>

#include "common.cuh"
#include "fgp2.h"
#include "pairwise.cuh"
#include "prox_args.cuh"

namespace bsgd {

namespace cg = cooperative_groups;

namespace {

constexpr int kF2K = 5;          // sums of the dual pass
constexpr int kF2MaxCtas = 128;
constexpr int kF2MaxThreads = 512;

struct Col2 {
    double x, y;
};

__device__ __forceinline__ Col2 ld2(const double *p) {
    const double2 v = *reinterpret_cast<const double2 *>(p);
    return {v.x, v.y};
}
__device__ __forceinline__ Col2 ldg2(const double *p) {
    const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    return {v.x, v.y};
}
__device__ __forceinline__ void st2(double *p, double x, double y) {
    *reinterpret_cast<double2 *>(p) = make_double2(x, y);
}

// ((down - here_v) + right) - here_h (tv.py:124-132, divergence), zero terms passed as 0.0
__device__ __forceinline__ double div4(double down, double here_v, double right, double here_h) {
    return rn_sub(rn_add(rn_sub(down, here_v), right), here_h);
}

// c / max(|c|, 1) (tv.py:211-214).  Inside the unit ball (m2 < 1) sqrt(m2) <= 1,
// so the divisor is exactly 1.0 and c / 1.0 == c bit for bit: the sqrt and the
// two IEEE divisions run only where the projection is active (NaN takes the
// division path, as np.maximum propagates it).
__device__ __forceinline__ void proj2(double &cv, double &ch) {
    const double m2 = rn_add(rn_mul(cv, cv), rn_mul(ch, ch));
    if (!(m2 < 1.0)) {
        double mag = sqrt(m2);
        mag = (mag < 1.0) ? 1.0 : mag;
        cv = cv / mag;
        ch = ch / mag;
    }
}

struct F2 {
    int W, H, R, r0, r1;
    int tau, t0, lane, warp, nw;
    double w, step;
    const double *b;
    double *stage;   // [2][kF2K][W]
    double *leafv;   // [R * W / 128][kF2K]
    double *uxch;    // [2][nw]  lane 31's u (left neighbour of the next warp's lane 0)
    double *cxch;    // [2][nw]  lane 0's ch (right neighbour of the previous warp's lane 31)
};

// Row s's staged terms -> leaf sums in numpy order (8-lane groups, 16 strided
// terms per accumulator), written to leafv[(s - r0) * W/128 + leaf][k].
template <int K>
__device__ __forceinline__ void f2_reduce_row(const F2 &f, const double *stage, int srow) {
    const int per_k = f.W >> 4;             // (W / 128 leaves) x 8 accumulators
    const int i = threadIdx.x;
    if (i < per_k * K) {
        const int k = i / per_k, rem = i - k * per_k;
        const int leaf = rem >> 3, j = rem & 7;
        const double *src = stage + (size_t)k * f.W + leaf * 128 + j;
        double acc = src[0];
#pragma unroll
        for (int q = 1; q < 16; ++q) acc = rn_add(acc, src[8 * q]);
        const unsigned gm = 0xFFu << (f.lane & 24);
        acc = rn_add(acc, __shfl_xor_sync(gm, acc, 1, 8));
        acc = rn_add(acc, __shfl_xor_sync(gm, acc, 2, 8));
        acc = rn_add(acc, __shfl_xor_sync(gm, acc, 4, 8));
        if (j == 0) f.leafv[((size_t)srow * (f.W >> 7) + leaf) * K + k] = acc;
    }
}

// CTA leaf values -> part[blockIdx.x] (warp k folds sum k), grid barrier, and the
// G CTA results combined the same way; every thread gets the numpy-order totals.
template <int K>
__device__ __forceinline__ void f2_finish_sum(cg::grid_group &grid, const F2 &f, double *red, int &round,
                                              int ds, double (&out)[K]) {
    double *buf = red + (size_t)(round & 1) * kMaxPartials * kPwMaxK;
    (void)ds;
    __syncthreads();
    const int Q = f.R * (f.W >> 7);
    for (int k = f.warp; k < K; k += f.nw) {
        const double v = warp_pw_tree<K, false>(f.leafv + k, Q, f.lane);
        if (f.lane == 0) buf[(size_t)blockIdx.x * K + k] = v;
    }
    grid.sync();
    for (int k = f.warp; k < K; k += f.nw) {
        const double v = warp_pw_tree<K, true>(buf + k, (int)gridDim.x, f.lane);
        if (f.lane == 0) f.stage[k] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) out[k] = f.stage[k];
    __syncthreads();
    ++round;
}

// One fused candidate + dual-value + commit pass (see the header).  src: the
// point the candidate steps from (q, or p on a restart); szero / pzero: the
// field is identically zero (first iteration; read as literal zeros).  Every
// global load of a step is issued before its arithmetic.
__device__ __forceinline__ void f2_pass(const F2 &f, double *fb, int fs, int iS, bool szero, int iP, bool pzero,
                                        double beta, int iC, int iQ) {
    const int W = f.W, H = f.H, t0 = f.t0, lane = f.lane, warp = f.warp;
    const double *Sv = fb + iS * fs, *Sh = Sv + fs, *Pv = fb + iP * fs, *Ph = Pv + fs;
    double *Cv = fb + iC * fs, *Ch = Cv + fs, *Qv = fb + iQ * fs, *Qh = Qv + fs;
    const bool has_left = t0 > 0, has_right = t0 + 2 < W;
    Col2 qvH{0.0, 0.0}, qvC{0.0, 0.0}, qhC{0.0, 0.0};
    Col2 um{0.0, 0.0}, uc{0.0, 0.0};
    Col2 bC{0.0, 0.0}, bB{0.0, 0.0};
    Col2 cpv{0.0, 0.0}, cph{0.0, 0.0};   // c(s_b)
    const int kstart = f.r0 == 0 ? 1 : 0;
    {
        const int s_first = f.r0 == 0 ? 0 : f.r0 - 1;
        if (!szero) qvH = ld2(Sv + s_first * W + t0);
    }
    for (int k = kstart; k <= f.R + 2; ++k) {
        const int su = f.r0 - 1 + k, sc = su - 1, sb = su - 2;
        const bool u_on = su <= f.r1 && su < H;
        const bool c_on = sc >= f.r0 && sc <= f.r1 && sc < H;
        const bool b_on = sb >= f.r0 && sb < f.r1;
        const int ou = su * W + t0, ob = sb * W + t0;
        // ---- loads of the step ----
        Col2 qvN{0.0, 0.0}, qhU{0.0, 0.0}, bU{0.0, 0.0}, pv{0.0, 0.0}, ph{0.0, 0.0};
        double qhR = 0.0;
        if (u_on) {
            if (!szero) {
                if (su + 1 < H) qvN = ld2(Sv + ou + W);
                qhU = ld2(Sh + ou);
                if (lane == 31 && has_right) qhR = Sh[ou + 2];
            }
            bU = ldg2(f.b + ou);
        }
        if (b_on && !pzero) {
            pv = ld2(Pv + ob);
            ph = ld2(Ph + ob);
        }
        // the previous row's leaf sums, while this step's loads are in flight
        if (sb - 1 >= f.r0 && sb - 1 < f.r1) f2_reduce_row<kF2K>(f, f.stage + ((sb - 1) & 1) * kF2K * W, sb - 1 - f.r0);
        // ---- U: u(su) ----
        Col2 un{0.0, 0.0};
        if (u_on) {
            const double sh = __shfl_down_sync(0xffffffffu, qhU.x, 1);
            if (lane != 31) qhR = sh;
            const double hv0 = su > 0 ? qvH.x : 0.0, hv1 = su > 0 ? qvH.y : 0.0;
            un.x = rn_add(bU.x, rn_mul(f.w, div4(qvN.x, hv0, qhU.y, has_left ? qhU.x : 0.0)));
            un.y = rn_add(bU.y, rn_mul(f.w, div4(qvN.y, hv1, has_right ? qhR : 0.0, qhU.y)));
            if (lane == 31) f.uxch[(su & 1) * f.nw + warp] = un.y;
        }
        // ---- C: c(sc) ----
        Col2 cnv{0.0, 0.0}, cnh{0.0, 0.0};
        if (c_on) {
            double uleft = __shfl_up_sync(0xffffffffu, uc.y, 1);
            if (lane == 0) uleft = warp > 0 ? f.uxch[(sc & 1) * f.nw + warp - 1] : 0.0;
            const double gv0 = sc > 0 ? rn_sub(uc.x, um.x) : 0.0;
            const double gv1 = sc > 0 ? rn_sub(uc.y, um.y) : 0.0;
            const double gh0 = has_left ? rn_sub(uc.x, uleft) : 0.0;
            const double gh1 = rn_sub(uc.y, uc.x);
            cnv.x = rn_add(qvC.x, rn_mul(f.step, gv0));
            cnh.x = rn_add(qhC.x, rn_mul(f.step, gh0));
            cnv.y = rn_add(qvC.y, rn_mul(f.step, gv1));
            cnh.y = rn_add(qhC.y, rn_mul(f.step, gh1));
            proj2(cnv.x, cnh.x);
            proj2(cnv.y, cnh.y);
            if (lane == 0) f.cxch[(sc & 1) * f.nw + warp] = cnh.x;
        }
        // ---- B: terms, commit and c of row sb ----
        if (b_on) {
            double right1 = __shfl_down_sync(0xffffffffu, cph.x, 1);
            if (lane == 31) right1 = warp + 1 < f.nw ? f.cxch[(sb & 1) * f.nw + warp + 1] : 0.0;
            const bool down = sb + 1 < H;
            const double d0 = div4(down ? cnv.x : 0.0, sb > 0 ? cpv.x : 0.0, cph.y, has_left ? cph.x : 0.0);
            const double d1 = div4(down ? cnv.y : 0.0, sb > 0 ? cpv.y : 0.0, has_right ? right1 : 0.0, cph.y);
            const double res0 = rn_add(bB.x, rn_mul(f.w, d0)), res1 = rn_add(bB.y, rn_mul(f.w, d1));
            const double sv0 = rn_sub(cpv.x, pv.x), sv1 = rn_sub(cpv.y, pv.y);
            const double sh0 = rn_sub(cph.x, ph.x), sh1 = rn_sub(cph.y, ph.y);
            st2(Qv + ob, rn_add(cpv.x, rn_mul(beta, sv0)), rn_add(cpv.y, rn_mul(beta, sv1)));
            st2(Qh + ob, rn_add(cph.x, rn_mul(beta, sh0)), rn_add(cph.y, rn_mul(beta, sh1)));
            st2(Cv + ob, cpv.x, cpv.y);
            st2(Ch + ob, cph.x, cph.y);
            double *stg = f.stage + (sb & 1) * kF2K * W + t0;
            st2(stg, rn_mul(res0, res0), rn_mul(res1, res1));
            st2(stg + W, rn_mul(sv0, sv0), rn_mul(sv1, sv1));
            st2(stg + 2 * W, rn_mul(sh0, sh0), rn_mul(sh1, sh1));
            st2(stg + 3 * W, rn_mul(cpv.x, cpv.x), rn_mul(cpv.y, cpv.y));
            st2(stg + 4 * W, rn_mul(cph.x, cph.x), rn_mul(cph.y, cph.y));
        }
        __syncthreads();
        // ---- roll ----
        um = uc;
        uc = un;
        qvC = qvH;
        qhC = qhU;
        qvH = qvN;
        cpv = cnv;
        cph = cnh;
        bB = bC;
        bC = bU;
    }
    // the last row's leaf sums (its terms were staged before the final barrier)
    f2_reduce_row<kF2K>(f, f.stage + ((f.r1 - 1) & 1) * kF2K * W, f.R - 1);
}

// out(s, t) = b + w div p (tv.py:250)
__device__ __forceinline__ double f2_out_at(const F2 &f, const double *Pv, const double *Ph, int s, int t) {
    const size_t o = (size_t)s * f.W + t;
    const double down = s + 1 < f.H ? Pv[o + f.W] : 0.0;
    const double hv = s > 0 ? Pv[o] : 0.0;
    const double right = t + 1 < f.W ? Ph[o + 1] : 0.0;
    const double hh = t > 0 ? Ph[o] : 0.0;
    return rn_add(__ldg(f.b + o), rn_mul(f.w, div4(down, hv, right, hh)));
}

__device__ __forceinline__ double tv2(double uc, double up, double ul, bool has_up, bool has_left) {
    const double dv = has_up ? rn_sub(uc, up) : 0.0;
    const double dh = has_left ? rn_sub(uc, ul) : 0.0;
    return sqrt(rn_add(rn_mul(dv, dv), rn_mul(dh, dh)));
}

__global__ void __launch_bounds__(kF2MaxThreads, 1) fgp2_rows_kernel(ProxArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double dsm[];
    F2 f;
    f.W = (int)a.W;
    f.H = (int)a.H;
    f.R = f.H / (int)gridDim.x;
    f.r0 = (int)blockIdx.x * f.R;
    f.r1 = f.r0 + f.R;
    f.tau = threadIdx.x;
    f.t0 = 2 * f.tau;
    f.lane = threadIdx.x & 31;
    f.warp = threadIdx.x >> 5;
    f.nw = (int)blockDim.x >> 5;
    f.w = a.w;
    f.step = a.step;
    f.b = a.b;
    f.stage = dsm;
    f.leafv = f.stage + 2 * kF2K * f.W;
    f.uxch = f.leafv + (size_t)f.R * (f.W >> 7) * kF2K;
    f.cxch = f.uxch + 2 * f.nw;
    const int W = f.W, H = f.H, t0 = f.t0, lane = f.lane;
    const bool has_left = t0 > 0, has_right = t0 + 2 < W;
    int round = 0;

    // --- setup: phi_prev = np.sum(b*b) (tv.py:203), TV(b) for the fallback test (tv.py:251)
    double v2[2];
    {
        Col2 bprev{0.0, 0.0};
        if (f.r0 > 0) bprev = ldg2(f.b + (size_t)(f.r0 - 1) * W + t0);
        for (int s = f.r0; s < f.r1; ++s) {
            const size_t o = (size_t)s * W + t0;
            const Col2 bb = ldg2(f.b + o);
            double bl = __shfl_up_sync(0xffffffffu, bb.y, 1);
            if (lane == 0) bl = has_left ? __ldg(f.b + o - 1) : 0.0;
            double *stg = f.stage + (size_t)(s & 1) * kF2K * W + t0;
            st2(stg, rn_mul(bb.x, bb.x), rn_mul(bb.y, bb.y));
            st2(stg + W, tv2(bb.x, bprev.x, bl, s > 0, has_left), tv2(bb.y, bprev.y, bb.x, s > 0, true));
            __syncthreads();
            f2_reduce_row<2>(f, f.stage + (size_t)(s & 1) * kF2K * W, s - f.r0);
            bprev = bb;
        }
        f2_finish_sum<2>(grid, f, a.red, round, a.ds, v2);
    }
    double phi_prev = v2[0];
    const double tv_b = v2[1];
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.dual != nullptr) a.dual[0] = phi_prev;

    // fields f[k] = fb + k * fs: p, q, c, q' at 0 / 2 / 4 / 6 (parity 0); every accepted
    // iteration swaps p <-> c and q <-> q' (parity flip)
    double *fb = a.f[0];
    const int fs = (int)(a.f[1] - a.f[0]);
    int par = 0;
    bool zero = true;   // p = q = 0 before the first iteration (tv.py:198-201)
    double t_mom = 1.0;
    int iters = 0, restarts = 0, converged = 0;
    for (int it = 0; it < a.max_iters; ++it) {
        double t_next = 0.5 * (1.0 + sqrt(rn_add(1.0, rn_mul(rn_mul(4.0, t_mom), t_mom))));
        double beta = (t_mom - 1.0) / t_next;
        double vc[kF2K];
        const int iP = par ? 4 : 0, iC = par ? 0 : 4, iQ = par ? 6 : 2, iQn = par ? 2 : 6;
        f2_pass(f, fb, fs, iQ, zero, iP, zero, beta, iC, iQn);
        f2_finish_sum<kF2K>(grid, f, a.red, round, a.ds, vc);
        double phi = vc[0];
        if (phi > phi_prev) {  // restart from the last accepted point (tv.py:217-231)
            ++restarts;
            t_mom = 1.0;
            t_next = 0.5 * (1.0 + sqrt(rn_add(1.0, rn_mul(rn_mul(4.0, t_mom), t_mom))));
            beta = (t_mom - 1.0) / t_next;
            f2_pass(f, fb, fs, iP, zero, iP, zero, beta, iC, iQn);
            f2_finish_sum<kF2K>(grid, f, a.red, round, a.ds, vc);
            phi = vc[0];
        }
        par ^= 1;       // p <- c, q <- q'
        zero = false;
        phi_prev = (phi_prev < phi) ? phi_prev : phi;  // Python min(phi, phi_prev)
        t_mom = t_next;
        iters = it + 1;
        if (blockIdx.x == 0 && threadIdx.x == 0 && a.dual != nullptr) a.dual[it + 1] = phi_prev;
        const double change = sqrt(rn_add(vc[1], vc[2])), scale = sqrt(rn_add(vc[3], vc[4]));
        const double floor_scale = (1e-30 > scale) ? 1e-30 : scale;  // Python max(scale, 1e-30)
        if (change <= a.tol * floor_scale) {
            converged = 1;
            break;
        }
    }

    // --- finalize: out = b + w div p (tv.py:250) into scratch, the primal energies
    //     ||out - b||^2 and TV(out) (tv.py:166-169) in numpy order
    double *tmp = fb + (par ? 0 : 4) * fs;   // c's first field: scratch once p is final
    double e2[2];
    {
        const double *Pv = fb + (par ? 4 : 0) * fs, *Ph = Pv + fs;
        Col2 oprev{0.0, 0.0};
        if (f.r0 > 0) {
            oprev.x = f2_out_at(f, Pv, Ph, f.r0 - 1, t0);
            oprev.y = f2_out_at(f, Pv, Ph, f.r0 - 1, t0 + 1);
        }
        for (int s = f.r0; s < f.r1; ++s) {
            const size_t o = (size_t)s * W + t0;
            const Col2 bb = ldg2(f.b + o);
            const Col2 ph = ld2(Ph + o);
            const Col2 pvh = ld2(Pv + o);
            Col2 pvd{0.0, 0.0};
            if (s + 1 < H) pvd = ld2(Pv + o + W);
            double phr = __shfl_down_sync(0xffffffffu, ph.x, 1);
            if (lane == 31) phr = has_right ? Ph[o + 2] : 0.0;
            Col2 out;
            out.x = rn_add(bb.x, rn_mul(f.w, div4(pvd.x, s > 0 ? pvh.x : 0.0, ph.y, has_left ? ph.x : 0.0)));
            out.y = rn_add(bb.y, rn_mul(f.w, div4(pvd.y, s > 0 ? pvh.y : 0.0, has_right ? phr : 0.0, ph.y)));
            st2(tmp + o, out.x, out.y);
            double ol = __shfl_up_sync(0xffffffffu, out.y, 1);
            if (lane == 0) ol = has_left ? f2_out_at(f, Pv, Ph, s, t0 - 1) : 0.0;
            const double d0 = rn_sub(out.x, bb.x), d1 = rn_sub(out.y, bb.y);
            double *stg = f.stage + (size_t)(s & 1) * kF2K * W + t0;
            st2(stg, rn_mul(d0, d0), rn_mul(d1, d1));
            st2(stg + W, tv2(out.x, oprev.x, ol, s > 0, has_left), tv2(out.y, oprev.y, out.x, s > 0, true));
            __syncthreads();
            f2_reduce_row<2>(f, f.stage + (size_t)(s & 1) * kF2K * W, s - f.r0);
            oprev = out;
        }
        f2_finish_sum<2>(grid, f, a.red, round, a.ds, e2);
    }
    const double two_w = 2.0 * a.w;
    const double obj_out = rn_add(e2[0], rn_mul(two_w, e2[1]));
    const double obj_b = rn_add(0.0, rn_mul(two_w, tv_b));
    const int fell = obj_out > obj_b ? 1 : 0;

    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    if (a.out_img != nullptr) {
        for (int s = f.r0; s < f.r1; ++s) {
            const size_t o = (size_t)s * W + t0;
            const Col2 v = fell ? ldg2(f.b + o) : ld2(tmp + o);
            st2(a.out_img + o, v.x, v.y);
        }
    } else {
        // epoch mode: x_next in vector order (a gather through perm, visible after the
        // energy pass's grid barrier) and the fused statistics of the step
        double st[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t k = tid; k < a.N; k += nthr) {
            const int64_t p = (a.perm != nullptr) ? a.perm[k] : k;
            const double xv = fell ? __ldg(f.b + p) : tmp[p];
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
        block_sum<4>(st, f.stage);
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

size_t f2_smem(int W, int R, int nw) {
    return sizeof(double) * ((size_t)2 * kF2K * W + (size_t)R * (W / 128) * kF2K + 4 * (size_t)nw);
}

int f2_grid(int64_t H) { return (int)(H < kF2MaxCtas ? H : kF2MaxCtas); }

}  // namespace

bool fgp2_rows_supported(const ProxArgs &a) {
    auto pow2 = [](int64_t v) { return v > 0 && (v & (v - 1)) == 0; };
    if (a.D > 1 || !pow2(a.W) || !pow2(a.H) || a.W < 128 || a.W > 2 * kF2MaxThreads) return false;
    if ((a.H / f2_grid(a.H)) * (a.W / 128) > 512) return false;   // leaves per CTA (warp_pw_tree)
    if ((reinterpret_cast<uintptr_t>(a.b) & 15) || (a.out_img && (reinterpret_cast<uintptr_t>(a.out_img) & 15)))
        return false;
    const int64_t fs = a.f[1] - a.f[0];
    if (fs < a.N || (fs & 1) || (reinterpret_cast<uintptr_t>(a.f[0]) & 15) || a.N + 8 * fs > INT32_MAX) return false;
    for (int k = 0; k < 8; ++k)
        if (a.f[k] != a.f[0] + k * fs) return false;   // one workspace, fixed field stride
    return true;
}

cudaError_t fgp2_rows_launch(const ProxArgs &a, int num_sms, cudaStream_t st) {
    const int W = (int)a.W, threads = W / 2;
    const int G = f2_grid(a.H);
    const int R = (int)(a.H / G);
    const size_t smem = f2_smem(W, R, (threads + 31) / 32);
    static int attr_set = 0;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(fgp2_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
        attr_set = 1;
    }
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fgp2_rows_kernel, threads, smem);
    if (e != cudaSuccess) return e;
    if ((int64_t)occ * num_sms < G) return cudaErrorCooperativeLaunchTooLarge;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fgp2_rows_kernel, a);
}

}  // namespace bsgd
