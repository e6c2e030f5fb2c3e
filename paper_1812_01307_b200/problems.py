"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference ships only a fan-beam / Shepp-Logan generator
(`pkg/src/bsgdtv/sim.py:150-283`); the benchmark configurations need a
parallel-beam Siddon projector, random-ellipse phantoms, absolute-sigma noise
and a random least-squares system, none of which exist upstream
(SURVEY.md §3.4, §8c "Inputs missing from the reference").  This module
builds them on the host, deterministically from explicit seeds, so the CUDA
path and the CPU oracle are always fed byte-identical A, y and x_true.

Conventions shared with the reference tracer (`sim.py:165-204`):
* the n x n image covers [-n/2, n/2]^2 in pixel units, row 0 at the top, so
  pixel (s, t) has row-major index s*n + t;
* matrix entries are exact ray/pixel intersection lengths (pixel pitch 1);
* rows are ordered angle-major, then detector bin.

Generation is setup work, not the hot path: it runs once per problem and is
never timed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy import sparse

# --- phantoms -----------------------------------------------------------


def ellipse_parameters(num_ellipses: int, seed: int) -> np.ndarray:
    """(k, 6) array: centre x, centre y, semi-axis a, semi-axis b, angle, intensity.

    Centres are uniform in the unit disc, semi-axes U[0.05, 0.4], rotation
    U[0, pi), additive intensity U[0, 1] (BASELINE.json configs[0]).
    """
    rng = np.random.default_rng(seed)
    u = rng.random((num_ellipses, 6))
    rad = np.sqrt(u[:, 0])
    ang = 2.0 * math.pi * u[:, 1]
    out = np.empty_like(u)
    out[:, 0] = rad * np.cos(ang)
    out[:, 1] = rad * np.sin(ang)
    out[:, 2] = 0.05 + 0.35 * u[:, 2]
    out[:, 3] = 0.05 + 0.35 * u[:, 3]
    out[:, 4] = math.pi * u[:, 4]
    out[:, 5] = u[:, 5]
    return out


def ellipse_phantom(n: int, num_ellipses: int, seed: int) -> np.ndarray:
    """Random-ellipse phantom rasterised at pixel centres, shape (n, n), float64.

    Normalised coordinates follow `sim.py:111-113`: column centres
    (2t + 1 - n)/n, row centres (n - 2s - 1)/n.
    """
    params = ellipse_parameters(num_ellipses, seed)
    cols = (2.0 * np.arange(n) + 1.0 - n) / n
    rows = (n - 2.0 * np.arange(n) - 1.0) / n
    xu, yu = np.meshgrid(cols, rows)
    img = np.zeros((n, n))
    for cx, cy, a, b, phi, val in params:
        ct, st = math.cos(phi), math.sin(phi)
        xr = (xu - cx) * ct + (yu - cy) * st
        yr = -(xu - cx) * st + (yu - cy) * ct
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += val
    return img


def ellipsoid_parameters(num_ellipsoids: int, seed: int) -> np.ndarray:
    """(k, 8): centre x, y, z, semi-axes a, b, c, rotation about z, intensity.

    3-D analogue of `ellipse_parameters` for configs[4] ("3D random ellipsoids
    (40, seeded)"): centres uniform in the unit ball, semi-axes U[0.05, 0.4],
    in-plane rotation U[0, pi), additive intensity U[0, 1].
    """
    rng = np.random.default_rng(seed)
    u = rng.random((num_ellipsoids, 8))
    rad = np.cbrt(u[:, 0])
    cos_pol = 2.0 * u[:, 1] - 1.0
    sin_pol = np.sqrt(np.maximum(0.0, 1.0 - cos_pol * cos_pol))
    az = 2.0 * math.pi * u[:, 2]
    out = np.empty_like(u)
    out[:, 0] = rad * sin_pol * np.cos(az)
    out[:, 1] = rad * sin_pol * np.sin(az)
    out[:, 2] = rad * cos_pol
    out[:, 3:6] = 0.05 + 0.35 * u[:, 3:6]
    out[:, 6] = math.pi * u[:, 6]
    out[:, 7] = u[:, 7]
    return out


def ellipsoid_phantom(n: int, depth: int, num_ellipsoids: int, seed: int) -> np.ndarray:
    """Random-ellipsoid phantom at voxel centres, shape (depth, n, n), float64.

    In-plane coordinates as `ellipse_phantom`; slice z sits at (2z + 1 - depth)/depth.
    """
    params = ellipsoid_parameters(num_ellipsoids, seed)
    cols = (2.0 * np.arange(n) + 1.0 - n) / n
    rows = (n - 2.0 * np.arange(n) - 1.0) / n
    zs = (2.0 * np.arange(depth) + 1.0 - depth) / depth
    xu, yu = np.meshgrid(cols, rows)
    vol = np.zeros((depth, n, n))
    for cx, cy, cz, a, b, c, phi, val in params:
        ct, st = math.cos(phi), math.sin(phi)
        xr = (xu - cx) * ct + (yu - cy) * st
        yr = -(xu - cx) * st + (yu - cy) * ct
        plane = (xr / a) ** 2 + (yr / b) ** 2
        for z in range(depth):
            dz = ((zs[z] - cz) / c) ** 2
            if dz <= 1.0:
                vol[z][plane + dz <= 1.0] += val
    return vol


def interleaved_perm(n_pixels: int, depth: int) -> np.ndarray:
    """Solver position k = pixel*depth + z  ->  z-major voxel z*n_pixels + pixel."""
    k = np.arange(n_pixels * depth, dtype=np.int64)
    return (k % depth) * n_pixels + k // depth


# --- parallel-beam Siddon projector --------------------------------------


def _trace_angle(n: int, theta: float, offsets: np.ndarray):
    """Siddon traversal of every detector ray of one view, vectorised over rays.

    Ray k is p(t) = o_k (cos th, sin th) + t (-sin th, cos th).  Returns
    (ray ids, row-major pixel ids, lengths) for all nonzero intersections.
    """
    h = n / 2.0
    ct, st = math.cos(theta), math.sin(theta)
    px = offsets * ct
    py = offsets * st
    # directions within 1e-12 of an axis are snapped to it, so rays that run
    # along a grid line (cos(pi/2) = 6e-17) are traced like the exact axis case
    dx = 0.0 if abs(st) < 1e-12 else -st
    dy = 0.0 if abs(ct) < 1e-12 else ct
    nb = offsets.shape[0]
    t_lo = np.full(nb, -np.inf)
    t_hi = np.full(nb, np.inf)
    inside = np.ones(nb, dtype=bool)
    for p0, d in ((px, dx), (py, dy)):
        if d == 0.0:
            inside &= (p0 >= -h) & (p0 <= h)
        else:
            t1 = (-h - p0) / d
            t2 = (h - p0) / d
            t_lo = np.maximum(t_lo, np.minimum(t1, t2))
            t_hi = np.minimum(t_hi, np.maximum(t1, t2))
    inside &= (t_hi - t_lo) > 1e-12
    if not inside.any():
        return (np.empty(0, np.int64),) * 2 + (np.empty(0),)
    rays = np.nonzero(inside)[0]
    px, py, t_lo, t_hi = px[rays], py[rays], t_lo[rays], t_hi[rays]
    planes = np.arange(n + 1, dtype=np.float64) - h
    parts = [t_lo[:, None], t_hi[:, None]]
    for p0, d in ((px, dx), (py, dy)):
        if d != 0.0:
            t = (planes[None, :] - p0[:, None]) / d
            t[(t <= t_lo[:, None]) | (t >= t_hi[:, None])] = np.nan
            parts.append(t)
    ts = np.sort(np.concatenate(parts, axis=1), axis=1)  # NaN sorts last
    seg = np.diff(ts, axis=1)
    mid = 0.5 * (ts[:, :-1] + ts[:, 1:])
    keep = seg > 1e-12  # False for NaN
    r_idx, c_idx = np.nonzero(keep)
    lengths = seg[r_idx, c_idx]
    m = mid[r_idx, c_idx]
    ix = np.clip(np.floor(px[r_idx] + m * dx + h).astype(np.int64), 0, n - 1)
    iy = np.clip(np.floor(py[r_idx] + m * dy + h).astype(np.int64), 0, n - 1)
    pix = (n - 1 - iy) * n + ix
    return rays[r_idx].astype(np.int64), pix, lengths


def parallel_beam_matrix(n: int, num_angles: int, num_bins: int,
                         dtype=np.float64) -> sparse.csr_array:
    """Siddon intersection-length matrix, (num_angles*num_bins) x n^2 CSR.

    Angles are uniform over [0, pi); detector bins have unit pitch and are
    centred on the rotation axis.  Indices are sorted and duplicates summed
    (the `BlockOperator` canonical form, `blockops.py:124-126`).
    """
    offsets = (np.arange(num_bins, dtype=np.float64) - (num_bins - 1) / 2.0)
    rows, cols, vals = [], [], []
    for a in range(num_angles):
        theta = math.pi * a / num_angles
        ray, pix, lng = _trace_angle(n, theta, offsets)
        rows.append(ray + a * num_bins)
        cols.append(pix)
        vals.append(lng)
    coo = sparse.coo_array(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(num_angles * num_bins, n * n),
    )
    csr = sparse.csr_array(coo)
    csr.sum_duplicates()
    csr.sort_indices()
    if dtype != np.float64:
        csr = sparse.csr_array((csr.data.astype(dtype), csr.indices, csr.indptr), shape=csr.shape)
    return csr


# --- random least-squares system (configs[1]) -----------------------------


def random_sparse_system(rows: int, cols: int, nnz_per_row: int, seed: int,
                         dtype=np.float32) -> sparse.csr_array:
    """rows x cols CSR with exactly ``nnz_per_row`` distinct uniform columns per row.

    Values are N(0,1)/sqrt(nnz_per_row).  Duplicate columns inside a row are
    redrawn until every row is duplicate-free, so the result is deterministic
    for a given seed.
    """
    if nnz_per_row > cols:
        raise ValueError("nnz_per_row exceeds the column count")
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, cols, size=(rows, nnz_per_row), dtype=np.int64)
    idx.sort(axis=1)
    while True:
        dup_rows = np.nonzero((np.diff(idx, axis=1) == 0).any(axis=1))[0]
        if dup_rows.size == 0:
            break
        fresh = rng.integers(0, cols, size=(dup_rows.size, nnz_per_row), dtype=np.int64)
        fresh.sort(axis=1)
        idx[dup_rows] = fresh
    vals = (rng.standard_normal((rows, nnz_per_row), dtype=np.float64)
            / math.sqrt(nnz_per_row)).astype(dtype)
    indptr = np.arange(0, rows * nnz_per_row + 1, nnz_per_row, dtype=np.int64)
    return sparse.csr_array((vals.ravel(), idx.astype(np.int32).ravel(), indptr), shape=(rows, cols))


# --- assembled problem instances ----------------------------------------


@dataclass
class ProblemData:
    """Host-side problem instance shared by the CUDA path and the oracle."""

    name: str
    matrix: sparse.csr_array        # canonical CSR (sorted, summed)
    y: np.ndarray                   # float64 measurements
    x_true: np.ndarray              # float64 ground truth (solver-vector order)
    height: int                     # image rows (1 for non-image problems)
    width: int
    num_row_blocks: int
    num_col_blocks: int
    lam: float
    max_inner_iters: int
    epochs: int
    seeds: dict

    @property
    def shape(self):
        return self.matrix.shape


def _matvec64(a: sparse.csr_array, x: np.ndarray) -> np.ndarray:
    return sparse.csr_array((a.data.astype(np.float64), a.indices, a.indptr), shape=a.shape) @ x


def ct_problem(name: str, n: int, num_angles: int, num_bins: int, num_ellipses: int,
               noise_frac: float, num_blocks: int, lam: float, max_inner_iters: int,
               epochs: int, dtype=np.float64, phantom_seed: int = 0,
               noise_seed: int = 1) -> ProblemData:
    """2D parallel-beam CT instance: y = A x_true + N(0, (noise_frac*max(A x_true))^2)."""
    a = parallel_beam_matrix(n, num_angles, num_bins, dtype=dtype)
    x_true = ellipse_phantom(n, num_ellipses, phantom_seed).ravel()
    clean = _matvec64(a, x_true)
    sigma = noise_frac * float(np.max(clean))
    noise = np.random.default_rng(noise_seed).standard_normal(clean.shape[0]) * sigma
    return ProblemData(name, a, clean + noise, x_true, n, n, num_blocks, num_blocks, lam,
                       max_inner_iters, epochs,
                       {"phantom": phantom_seed, "noise": noise_seed, "solver": 0})


def ls_problem(name: str, rows: int, cols: int, nnz_per_row: int, num_blocks: int,
               epochs: int, matrix_seed: int = 2, x_seed: int = 0,
               dtype=np.float32) -> ProblemData:
    """Noise-free random least-squares instance y = A x_true (lambda = 0)."""
    a = random_sparse_system(rows, cols, nnz_per_row, matrix_seed, dtype=dtype)
    x_true = np.random.default_rng(x_seed).standard_normal(cols)
    y = _matvec64(a, x_true)
    return ProblemData(name, a, y, x_true, 1, cols, num_blocks, num_blocks, 0.0, 20, epochs,
                       {"matrix": matrix_seed, "x_true": x_seed, "solver": 0})


def config(index: int, scale: float = 1.0) -> ProblemData:
    """BASELINE.json configs[index] (0-based), optionally shrunk for parity tests.

    ``scale`` < 1 shrinks the image side / system size while keeping the
    aspect ratios, sparsity, blocking and solver settings of the config.
    """
    if index == 0:
        n = max(16, int(round(128 * scale)))
        ang = max(8, int(round(180 * scale)))
        nb = max(9, int(round(183 * scale)) | 1)
        return ct_problem("C1", n, ang, nb, 10, 0.01, 4, 0.02, 20, 100, np.float64)
    if index == 1:
        rows = max(64, int(round(2_000_000 * scale)))
        cols = max(16, int(round(500_000 * scale)))
        return ls_problem("C2", rows, cols, min(32, cols), 8, 200)
    if index == 2:
        n = max(16, int(round(512 * scale)))
        ang = max(8, int(round(720 * scale)))
        nb = max(9, int(round(727 * scale)) | 1)
        return ct_problem("C3", n, ang, nb, 30, 0.005, 8, 0.01, 20, 100, np.float32)
    if index == 3:
        n = max(16, int(round(1024 * scale)))
        ang = max(8, int(round(1440 * scale)))
        nb = max(9, int(round(1449 * scale)) | 1)
        return ct_problem("C4", n, ang, nb, 60, 0.005, 8, 0.01, 20, 50, np.float32)
    raise ValueError(f"config index {index} has no host generator (3D config needs the device generator)")


# --- device-generated instances (configs[3]-size) -------------


@dataclass
class DeviceProblem:
    """CT instance whose projector lives only on the GPU (no host CSR)."""

    name: str
    op: object                      # blockops.BlockOperator built by from_parallel_beam
    y: np.ndarray                   # float64 measurements (host copy, rows doubles)
    x_true: np.ndarray
    height: int
    width: int
    num_row_blocks: int
    num_col_blocks: int
    lam: float
    max_inner_iters: int
    epochs: int
    seeds: dict
    depth: int = 1                  # > 1: slice-stacked volume (solver order interleaved, see layout())

    def layout(self, slice_major: bool = False):
        """Pixel / voxel layout of the solver vector (tv.PixelLayout or tv.VolumeLayout).

        Stacked volumes: by default the interleaved solver vector is itself the
        C-order (rows, columns, slices) volume, so the 3-D prox needs no
        permutation (isotropic TV does not depend on which axis is called z;
        only the rounding order of its sums does).  ``slice_major=True`` gives
        the (slices, rows, columns) view through `interleaved_perm` instead.
        """
        from . import tv
        if self.depth > 1:
            if slice_major:
                return tv.VolumeLayout(self.depth, self.height, self.width,
                                       interleaved_perm(self.height * self.width, self.depth))
            return tv.VolumeLayout.z_major(self.height, self.width, self.depth)
        return tv.PixelLayout.row_major(self.height, self.width)


def ct_problem_device(name: str, n: int, num_angles: int, num_bins: int, num_ellipses: int, noise_frac: float,
                      num_blocks: int, lam: float, max_inner_iters: int, epochs: int, dtype=np.float32,
                      phantom_seed: int = 0, noise_seed: int = 1, device=None) -> DeviceProblem:
    """Same instance definition as `ct_problem`, with A generated and kept on the GPU.

    y = A x_true is formed by the device SpMV (float64 accumulation), so it may
    differ from the host path's scipy product in the last bits; the noise draw
    is the same seeded numpy stream.
    """
    from .blockops import BlockOperator
    op = BlockOperator.from_parallel_beam(n, num_angles, num_bins, num_blocks, num_blocks, dtype=dtype,
                                          device=device)
    x_true = ellipse_phantom(n, num_ellipses, phantom_seed).ravel()
    clean = op.matvec(x_true, charge=False)
    sigma = noise_frac * float(np.max(clean))
    noise = np.random.default_rng(noise_seed).standard_normal(clean.shape[0]) * sigma
    return DeviceProblem(name, op, clean + noise, x_true, n, n, num_blocks, num_blocks, lam, max_inner_iters,
                         epochs, {"phantom": phantom_seed, "noise": noise_seed, "solver": 0})


def stacked_ct_problem_device(name: str, n: int, depth: int, num_angles: int, num_bins: int, num_ellipsoids: int,
                              noise_frac: float, num_blocks: int, lam: float, max_inner_iters: int, epochs: int,
                              dtype=np.float32, phantom_seed: int = 0, noise_seed: int = 1,
                              device=None) -> DeviceProblem:
    """3-D slice-stacked parallel-beam CT (configs[4]): A = A2 (x) I_depth on the GPU.

    x_true is the ellipsoid phantom in the interleaved solver order (voxel
    (z, s, t) at position (s*n + t)*depth + z); y = A x_true + N(0, sigma^2),
    sigma = noise_frac * max(A x_true).
    """
    from .blockops import BlockOperator
    op = BlockOperator.from_parallel_beam(n, num_angles, num_bins, num_blocks, num_blocks, dtype=dtype,
                                          device=device, depth=depth)
    vol = ellipsoid_phantom(n, depth, num_ellipsoids, phantom_seed)
    x_true = np.ascontiguousarray(vol.reshape(depth, n * n).T).ravel()
    clean = op.matvec(x_true, charge=False)
    sigma = noise_frac * float(np.max(clean))
    noise = np.random.default_rng(noise_seed).standard_normal(clean.shape[0]) * sigma
    return DeviceProblem(name, op, clean + noise, x_true, n, n, num_blocks, num_blocks, lam, max_inner_iters,
                         epochs, {"phantom": phantom_seed, "noise": noise_seed, "solver": 0}, depth=depth)


# 2-D CT configurations: name, image side, angles, bins, ellipses, noise fraction,
# blocks, lambda, FGP cap, epochs, value dtype (BASELINE.json configs[0], [2], [3])
CT_TABLE = {0: ("C1", 128, 180, 183, 10, 0.01, 4, 0.02, 20, 100, np.float64),
            2: ("C3", 512, 720, 727, 30, 0.005, 8, 0.01, 20, 100, np.float32),
            3: ("C4", 1024, 1440, 1449, 60, 0.005, 8, 0.01, 20, 50, np.float32)}


def config_device(index: int, scale: float = 1.0, device=None) -> DeviceProblem:
    """configs[0], [2], [3] or [4] with the projector generated on the GPU."""
    if index == 4:
        n = max(16, int(round(256 * scale)))
        depth = max(2, int(round(256 * scale)))
        ang = max(8, int(round(360 * scale)))
        nb = max(9, int(round(363 * scale)) | 1)
        return stacked_ct_problem_device("C5", n, depth, ang, nb, 40, 0.01, 16, 0.01, 10, 30, np.float32,
                                         device=device)
    if index not in CT_TABLE:
        raise ValueError(f"config index {index} is not a 2D CT configuration")
    name, n, ang, nb, ell, noise, blocks, lam, inner, epochs, dt = CT_TABLE[index]
    n = max(16, int(round(n * scale)))
    ang = max(8, int(round(ang * scale)))
    nb = max(9, int(round(nb * scale)) | 1)
    return ct_problem_device(name, n, ang, nb, ell, noise, blocks, lam, inner, epochs, dt, device=device)
