"""Step-size analysis (drop-in for `bsgdtv.spectral`, `spectral.py:25-123`).

`largest_eigenvalue` is the power iteration on A^T A that sets every
configuration's step (mu = 0.9 / (2 u_max)); here each iteration is two
device SpMVs (`bsgd_matvec` / `bsgd_rmatvec`) plus device dot products, with
the same seeded start vector, null-space restart and relative stop rule as
the reference (§8 f3: needed on the GPU where the CPU oracle cannot hold the
matrix).  The closed-form helpers are host arithmetic, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _native as nat
from .blockops import BlockOperator


class PowerIterationResult(NamedTuple):
    value: float
    converged: bool
    iterations: int


@dataclass(frozen=True)
class StepBound:
    """Largest eigenvalue of A^T A and the open step supremum 1/(2 u_max)."""

    u_max: float
    mu_sup: float

    def admits(self, mu: float) -> bool:
        return 0.0 < mu < self.mu_sup


def largest_eigenvalue(op: BlockOperator, tol: float = 1e-10, max_iters: int = 5000,
                       seed: int = 0) -> PowerIterationResult:
    """Power iteration for the largest eigenvalue of A^T A (`spectral.py:43-75`)."""
    if not tol > 0:
        raise ValueError("tol must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    t = nat.torch()
    rows, cols = op.shape
    dev = op.device
    rng = np.random.default_rng(seed)

    def fresh():
        v0 = rng.standard_normal(cols)
        v0 /= np.linalg.norm(v0)
        return nat.as_f64(v0, dev)

    v = fresh()
    av = t.empty(rows, dtype=t.float64, device=dev)
    atav = t.empty(cols, dtype=t.float64, device=dev)
    sc = t.empty(2, dtype=t.float64, device=dev)
    scratch = t.empty(nat.SCRATCH_BYTES // 8, dtype=t.float64, device=dev)
    st = nat.stream_ptr(dev)
    estimate = 0.0
    for k in range(1, max_iters + 1):
        op._charge(op.nnz)
        nat.call("bsgd_matvec", op.plan, nat.ptr(v), nat.ptr(av), st)
        nat.call("bsgd_dot", rows, nat.ptr(av), nat.ptr(av), nat.ptr(sc[0:1]), nat.ptr(scratch), st)
        op._charge(op.nnz)
        nat.call("bsgd_rmatvec", op.plan, nat.ptr(av), nat.ptr(atav), st)
        nat.call("bsgd_dot", cols, nat.ptr(atav), nat.ptr(atav), nat.ptr(sc[1:2]), nat.ptr(scratch), st)
        new_estimate, nrm2 = (float(x) for x in sc.cpu().tolist())
        norm = float(np.sqrt(nrm2))
        if norm == 0.0:
            v = fresh()
            continue
        v = atav / norm
        if k > 1 and abs(new_estimate - estimate) <= tol * max(new_estimate, 1e-300):
            return PowerIterationResult(new_estimate, True, k)
        estimate = new_estimate
    return PowerIterationResult(estimate, False, max_iters)


def step_bound(u_max: float) -> StepBound:
    if not u_max > 0:
        raise ValueError("u_max must be positive")
    return StepBound(u_max=float(u_max), mu_sup=1.0 / (2.0 * float(u_max)))


def iteration_eigenvalues(u: float, mu: float) -> tuple:
    """(1 +/- sqrt(1 - 8 mu u)) / 2 (`spectral.py:85-95`)."""
    root = np.sqrt(complex(1.0 - 8.0 * mu * u, 0.0))
    return complex((1.0 + root) / 2.0), complex((1.0 - root) / 2.0)


def predicted_spectral_radius(u_values, mu: float) -> float:
    radius = 0.0
    for u in np.asarray(u_values, dtype=np.float64):
        v1, v2 = iteration_eigenvalues(float(u), mu)
        radius = max(radius, abs(v1), abs(v2))
    return radius
