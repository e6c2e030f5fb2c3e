// Arguments of the TV prox kernels (fgp.cuh cooperative / split kernels,
// fgp2.cu row-walk kernel), shared by both translation units.
#pragma once

#include <stdint.h>

namespace bsgd {

constexpr int kProxFields = 10;   // workspace fields of the prox (fgp.cuh, fgp2.cu, slab.cuh)

struct ProxArgs {
    int64_t D, H, W, N;    // D = 1 for images; 3D volumes are z-major (z, row, column)
    const double *b;       // input image (row-major)
    double *f[kProxFields]; // p[DIM], q[DIM], c[DIM], u (workspace); 2D: pv, ph, qv, qh, cv, ch (+ q' for fgp2)
    double *red;           // [2][kMaxPartials * kPwMaxK] reduction partials
    double w, step, tol;
    int32_t max_iters;
    int32_t ds;            // numpy pairwise depth for N (pw_depth)
    int32_t fast;          // N == 128 * 2^ds: chunked fast path (pw_cta_fast)
    // outputs -- standalone (tv_prox) mode
    double *out_img;       // NULL in epoch mode
    // outputs -- epoch mode (vector order, fused statistics)
    double *x_next;
    const int64_t *perm;
    const double *x_k;
    const double *g;
    const double *x_true;
    double *xpart;         // [gridDim.x * 4] per-CTA statistics
    int64_t *nx;           // number of xpart rows written
    double *scal;          // [0] TV(final) [1] iterations [2] restarts [3] converged [4] fell_back
    int32_t *info;         // bsgd_prox_info or NULL
    double *dual;          // dual objectives or NULL
};

}  // namespace bsgd
