// Parallel-beam Siddon projector generated on the device.
//
// configs[3] (1024^2, 1440 x 1449 rays, ~1.9e9 nonzeros) and larger cannot be
// generated on the host in reasonable time or memory.  One thread traces one
// ray and emits its (pixel, intersection length) pairs directly into CSR
// storage; a first pass counts, an exclusive scan places rows.
//
// The arithmetic repeats paper_1812_01307_b200/problems.py::_trace_angle op
// for op with round-to-nearest intrinsics (no FMA), and cos/sin come from the
// host per angle, so the device matrix is bit-identical to the host one
// (tests/test_gpu_generator.py).  Crossing times of each axis are monotone in
// the plane index, so numpy's sort becomes a two-way merge; entries are then
// put in CSR column order by reversing monotone runs (the pixel row index and
// the pixel column index are both monotone along a ray).
#pragma once

#include <math.h>

#include "common.cuh"

namespace bsgd {

struct RayGeom {
    int64_t n;          // image side
    int64_t nbins;
    int64_t nrays;      // num_angles * nbins
    const double *ct;   // cos(theta_a), host-computed
    const double *st;   // sin(theta_a)
};

// traverse ray `ray`; Emit(pix, length) is called in traversal order
template <class Emit>
__device__ __forceinline__ void siddon_trace(const RayGeom &G, int64_t ray, Emit &emit, int &sig_s, int &sig_x) {
    const int64_t a = ray / G.nbins, b = ray - a * G.nbins;
    const double n = (double)G.n;
    const double h = n / 2.0;
    const double ct = G.ct[a], st = G.st[a];
    const double off = rn_sub((double)b, rn_sub((double)G.nbins, 1.0) / 2.0);
    const double px = rn_mul(off, ct), py = rn_mul(off, st);
    const double dx = (fabs(st) < 1e-12) ? 0.0 : -st;
    const double dy = (fabs(ct) < 1e-12) ? 0.0 : ct;
    sig_s = (dy > 0.0) ? -1 : ((dy < 0.0) ? 1 : 0);   // pixel row s = n-1-iy
    sig_x = (dx > 0.0) ? 1 : ((dx < 0.0) ? -1 : 0);
    double t_lo = -INFINITY, t_hi = INFINITY;
    bool inside = true;
    const double p0s[2] = {px, py}, ds[2] = {dx, dy};
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
        const double p0 = p0s[ax], d = ds[ax];
        if (d == 0.0) {
            inside = inside && (p0 >= -h) && (p0 <= h);
        } else {
            const double t1 = rn_sub(-h, p0) / d;
            const double t2 = rn_sub(h, p0) / d;
            t_lo = fmax(t_lo, fmin(t1, t2));
            t_hi = fmin(t_hi, fmax(t1, t2));
        }
    }
    if (!inside || !(rn_sub(t_hi, t_lo) > 1e-12)) return;
    // crossing times of the x / y planes k - h inside (t_lo, t_hi), each ascending
    auto tx = [&](int64_t k) { return rn_sub((double)k - h, px) / dx; };
    auto ty = [&](int64_t k) { return rn_sub((double)k - h, py) / dy; };
    int64_t kx = (dx > 0.0) ? 0 : G.n, kx_step = (dx > 0.0) ? 1 : -1, kx_left = (dx != 0.0) ? G.n + 1 : 0;
    int64_t ky = (dy > 0.0) ? 0 : G.n, ky_step = (dy > 0.0) ? 1 : -1, ky_left = (dy != 0.0) ? G.n + 1 : 0;
    auto next_x = [&](double &t) -> bool {
        while (kx_left > 0) {
            const double v = tx(kx);
            kx += kx_step;
            --kx_left;
            if (v > t_lo && v < t_hi) { t = v; return true; }
            if (!(v < t_hi)) { kx_left = 0; }
        }
        return false;
    };
    auto next_y = [&](double &t) -> bool {
        while (ky_left > 0) {
            const double v = ty(ky);
            ky += ky_step;
            --ky_left;
            if (v > t_lo && v < t_hi) { t = v; return true; }
            if (!(v < t_hi)) { ky_left = 0; }
        }
        return false;
    };
    double cx = 0.0, cy = 0.0;
    bool hx = next_x(cx), hy = next_y(cy);
    double prev = t_lo;
    const int64_t nm1 = G.n - 1;
    for (;;) {
        double cur;
        bool last = false;
        if (hx && (!hy || cx <= cy)) { cur = cx; hx = next_x(cx); }
        else if (hy) { cur = cy; hy = next_y(cy); }
        else { cur = t_hi; last = true; }
        const double seg = rn_sub(cur, prev);
        if (seg > 1e-12) {
            const double m = rn_mul(0.5, rn_add(prev, cur));
            int64_t ix = (int64_t)floor(rn_add(rn_add(px, rn_mul(m, dx)), h));
            int64_t iy = (int64_t)floor(rn_add(rn_add(py, rn_mul(m, dy)), h));
            ix = ix < 0 ? 0 : (ix > nm1 ? nm1 : ix);
            iy = iy < 0 ? 0 : (iy > nm1 ? nm1 : iy);
            emit((nm1 - iy) * G.n + ix, seg);
        }
        prev = cur;
        if (last) break;
    }
}

__global__ void siddon_count_kernel(RayGeom G, int64_t *counts) {
    for (int64_t ray = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ray < G.nrays;
         ray += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        int ss, sx;
        auto emit = [&](int64_t, double) { ++c; };
        siddon_trace(G, ray, emit, ss, sx);
        counts[ray] = c;
    }
}

template <typename V>
__global__ void siddon_fill_kernel(RayGeom G, const int64_t *indptr, int32_t *indices, V *vals) {
    for (int64_t ray = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ray < G.nrays;
         ray += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = indptr[ray];
        int64_t w = 0;
        int ss = 0, sx = 0;
        auto emit = [&](int64_t pix, double len) {
            indices[base + w] = (int32_t)pix;
            vals[base + w] = (V)len;
            ++w;
        };
        siddon_trace(G, ray, emit, ss, sx);
        if (w < 2) continue;
        auto rev = [&](int64_t lo, int64_t hi) {  // reverse [lo, hi)
            for (--hi; lo < hi; ++lo, --hi) {
                const int32_t ti = indices[base + lo]; indices[base + lo] = indices[base + hi]; indices[base + hi] = ti;
                const V tv = vals[base + lo]; vals[base + lo] = vals[base + hi]; vals[base + hi] = tv;
            }
        };
        // pixel row s is monotone along the ray: make it ascending
        if (ss < 0) rev(0, w);
        // pixel column ix is monotone along the ray: inside each row run make it ascending
        const int dir_x = (ss < 0) ? -sx : sx;
        if (dir_x < 0) {
            int64_t r0 = 0;
            const int64_t n = G.n;
            for (int64_t i = 1; i <= w; ++i) {
                if (i == w || indices[base + i] / n != indices[base + r0] / n) {
                    rev(r0, i);
                    r0 = i;
                }
            }
        }
    }
}

}  // namespace bsgd
