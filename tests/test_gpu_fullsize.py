"""Full-size parity at the stated epoch counts (north star: x within relative L2
1e-4 and objective within 1e-5 relative of the reference's CPU solver after
the configuration's epochs; identical matvec-unit tallies).

The CUDA path runs `run_solver` (`solvers.py:445-533`) through the drop-in
API; the checker is the CPU oracle (`oracle.run_bsgd`, pinned bit-exact to
the reference by tests/test_oracle_golden.py) on the identical A, y and mu:
mu comes from tests/golden/config_mu.json (computed once, tools/make_mu.py),
the CT matrices from the GPU generator copied to the host (bit-identical to
the host generator, tests/test_gpu_generator.py), y from the same instance.

    configs[1]: 2,000,000 x 500,000 random LS, 200 epochs, monitor on (defaults)
    configs[2]: 512^2 CT, lambda 0.01, FGP <= 20, 100 epochs, monitor on
    configs[3]: 1024^2 CT, 1.9e9 nonzeros, lambda 0.01, FGP <= 20, 50 epochs,
                monitor off (keeps the oracle's run to ~2 minutes on the box)
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

X_TOL = 1e-4
OBJ_TOL = 1e-5


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def mu_for(index):
    with open(os.path.join(GOLDEN, "config_mu.json")) as fh:
        return float(json.load(fh)[f"configs[{index}]"]["mu"])


def _compare(tr, ref):
    assert rel(tr.final_x, ref.final_x) < X_TOL
    got = np.array([tuple(s) for s in tr.samples])
    want = np.array(ref.samples)
    assert got.shape == want.shape
    assert np.array_equal(got[:, 0], want[:, 0])
    assert np.allclose(got[:, 2], want[:, 2], rtol=OBJ_TOL, atol=0)
    assert np.array_equal(got[:, 3], want[:, 3])             # matvec units, exactly
    ok = np.isfinite(want[:, 1])
    assert np.allclose(got[ok, 1], want[ok, 1], rtol=1e-5, atol=0)
    return got, want


def test_configs1_full_size_200_epochs(cuda_ok):
    from paper_1812_01307_b200 import blockops, problems, solvers
    d = problems.config(1)
    mu = mu_for(1)
    op = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, 8, 8))
    cfg = solvers.SolverConfig(mu=mu, epochs=200)
    tr = solvers.run_solver("bsgd", solvers.Problem(op, d.y, d.x_true), cfg, sample_every=20)
    del op
    oop = orc.OracleOperator(d.matrix, 8, 8)
    ref = orc.run_bsgd(oop, d.y, orc.Params(mu=mu, epochs=200), x_true=d.x_true, sample_every=20)
    _compare(tr, ref)
    assert list(tr.decrease_flags) == list(ref.decrease_flags)
    assert tr.relative_errors()[-1] < 1e-3


@pytest.mark.parametrize("index,epochs,monitor", [(2, 100, True), (3, 50, False)])
def test_ct_full_size_stated_epochs(cuda_ok, index, epochs, monitor):
    import torch
    from paper_1812_01307_b200 import problems, solvers, tv
    d = problems.config_device(index)
    assert d.epochs == epochs
    mu = mu_for(index)
    lay = d.layout()
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=epochs, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=monitor)
    tr = solvers.run_solver("bsgd", solvers.Problem(d.op, d.y, d.x_true, lay), cfg, sample_every=10)
    csr = d.op.tocsr()
    d.op._csr = None
    del d.op
    torch.cuda.empty_cache()
    oop = orc.OracleOperator(csr, 8, 8)
    prm = orc.Params(mu=mu, lam=d.lam, epochs=epochs, max_inner_iters=d.max_inner_iters, tol=1e-5,
                     monitor_decrease=monitor)
    ref = orc.run_bsgd(oop, d.y, prm, x_true=d.x_true, perm=np.arange(csr.shape[1]), hw=(d.height, d.width),
                       sample_every=10)
    _compare(tr, ref)
    if monitor:
        assert list(tr.decrease_flags) == list(ref.decrease_flags)
    # the prox ran and changed the iterate (lambda > 0): objective includes 2 lam TV(x)
    assert tr.objectives()[-1] < tr.objectives()[0]
    if index == 2:
        # the reference's own call -- BlockOperator(A_csr, partition) on the plain host CSR, no
        # grid hints: K1 finds the square image by itself and the plan infers the sinogram grid
        # of A^T's gathers from the matrix; the same run against the same oracle trace
        from paper_1812_01307_b200 import blockops
        op2 = blockops.BlockOperator(csr, blockops.make_partition(*csr.shape, 8, 8))
        ki = op2.kernel_info()
        assert ki["forward"] == "blocked_compressed" and ki["forward_order"] == "tile4"
        assert ki["transposed"] == "blocked_compressed" and ki["transposed_order"] == "tile8x2"
        tr2 = solvers.run_solver("bsgd", solvers.Problem(op2, d.y, d.x_true, lay), cfg, sample_every=10)
        _compare(tr2, ref)
        assert list(tr2.decrease_flags) == list(ref.decrease_flags)


def _kron_interleaved(a2, depth):
    from scipy import sparse
    a = sparse.csr_array(sparse.kron(sparse.csr_array(a2), sparse.identity(depth, format="csr"), format="csr"))
    a.sort_indices()
    return a


def test_configs4_shaped_30_epochs_vs_oracle(cuda_ok):
    """configs[4]-shaped (64^3 volume, 90 angles x 91 bins per slice, M = N = 16,
    lambda 0.01, 3-D TV FGP <= 10) for the configuration's 30 epochs through
    run_solver, against the oracle on the expanded kron(A2, I_D) CSR with the
    oracle's 3-D prox restatement: x bit-identical (the stacked kernels follow the
    reference's block-sequential order), objectives to 1e-12."""
    from paper_1812_01307_b200 import problems, solvers, spectral, tv
    d = problems.config_device(4, scale=0.25)
    assert (d.depth, d.height, d.num_row_blocks, d.epochs, d.max_inner_iters) == (64, 64, 16, 30, 10)
    mu = 0.9 / (2.0 * spectral.largest_eigenvalue(d.op, max_iters=50).value)
    lay = d.layout()
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=d.epochs, prox=tv.ProxSettings(d.max_inner_iters, 1e-5))
    tr = solvers.run_solver("bsgd", solvers.Problem(d.op, d.y, d.x_true, lay), cfg, sample_every=5)
    a2 = problems.parallel_beam_matrix(d.height, 90, 91, dtype=np.float32)
    a = _kron_interleaved(a2, d.depth)
    assert a.nnz == d.op.nnz
    oop = orc.OracleOperator(a, 16, 16)
    prm = orc.Params(mu=mu, lam=d.lam, epochs=d.epochs, max_inner_iters=d.max_inner_iters, tol=1e-5)
    ref = orc.run_bsgd(oop, d.y, prm, x_true=d.x_true, perm=lay.perm, hw=(lay.depth, lay.height, lay.width),
                       sample_every=5)
    assert np.array_equal(tr.final_x, ref.final_x)
    got, want = np.array([tuple(s) for s in tr.samples]), np.array(ref.samples)
    assert np.array_equal(got[:, 0], want[:, 0]) and np.array_equal(got[:, 3], want[:, 3])
    assert np.allclose(got[:, 2], want[:, 2], rtol=1e-12)
    assert list(tr.decrease_flags) == list(ref.decrease_flags)


def test_configs4_zslab_general_block_diagonal_csr(cuda_ok):
    """configs[4] as BASELINE.json states it -- a block-diagonal CSR per slice
    through the GENERAL BlockOperator(matrix) path -- on a z-slab of the
    configured size (16 of the 256 slices: 256^2 images, 360 x 363 rays,
    4.8e8 nonzeros, slice-major rows z * R2 + r), against the slice-stacked
    operator on the same slab: products to 1e-12 and three TV-regularised epochs
    (3-D prox, lambda 0.01) to 1e-10."""
    import torch
    from paper_1812_01307_b200 import blockops, problems, solvers, tv
    n, ang, nb, depth = 256, 360, 363, 16
    stk = blockops.BlockOperator.from_parallel_beam(n, ang, nb, 16, 16, dtype=np.float32, depth=depth)
    a2 = blockops.BlockOperator.from_parallel_beam(n, ang, nb, dtype=np.float32, tiles=False).tocsr()
    r2, c2, nnz2 = a2.shape[0], a2.shape[1], a2.nnz
    from scipy import sparse
    indptr = np.concatenate([a2.indptr[:-1] + z * nnz2 for z in range(depth)] + [[depth * nnz2]]).astype(np.int64)
    indices = np.concatenate([a2.indices + np.int32(z * c2) for z in range(depth)])
    data = np.tile(a2.data, depth)
    bd = sparse.csr_array((data, indices, indptr), shape=(depth * r2, depth * c2))
    gen = blockops.BlockOperator(bd, blockops.make_partition(*bd.shape, 16, 16))
    del bd, data, indices, indptr
    assert gen.nnz == stk.nnz == depth * nnz2
    assert all(gen.block_nnz(i, j) == (nnz2 if i == j else 0) for i in range(16) for j in range(16))
    # interleaved position k = pixel * depth + z  ->  slice-major index z * n_pixels + pixel
    rperm = problems.interleaved_perm(r2, depth)
    cperm = problems.interleaved_perm(c2, depth)

    def to_sm(v_int, perm):
        out = np.empty_like(v_int)
        out[perm] = v_int
        return out

    rng = np.random.default_rng(7)
    x_sm = rng.random(depth * c2)
    assert rel(gen.matvec(x_sm, charge=False), to_sm(stk.matvec(x_sm[cperm], charge=False), rperm)) < 1e-12
    w_sm = rng.standard_normal(depth * r2)
    assert rel(gen.rmatvec(w_sm, charge=False), to_sm(stk.rmatvec(w_sm[rperm], charge=False), cperm)) < 1e-12
    # three epochs of the solver on the same data through both operators
    xt_sm = problems.ellipsoid_phantom(n, depth, 40, 0).ravel()
    clean = stk.matvec(xt_sm[cperm], charge=False)
    y_int = clean + np.random.default_rng(1).standard_normal(clean.shape[0]) * 0.01 * float(np.max(clean))
    y_sm = to_sm(y_int, rperm)
    mu = mu_for(4)
    cfg = solvers.SolverConfig(mu=mu, lam=0.01, epochs=3, prox=tv.ProxSettings(10, 1e-5))
    st_g = solvers.init_bsgd_state(gen, y_sm, cfg)
    st_s = solvers.init_bsgd_state(stk, y_int, cfg)
    lay_g = tv.VolumeLayout.z_major(depth, n, n)
    lay_s = tv.VolumeLayout(depth, n, n, cperm)
    for _ in range(3):
        solvers.bsgd_tv_iteration(st_g, gen, y_sm, cfg, layout=lay_g)
        solvers.bsgd_tv_iteration(st_s, stk, y_int, cfg, layout=lay_s)
    torch.cuda.synchronize()
    assert rel(st_g.x, to_sm(st_s.x, cperm)) < 1e-10
    assert rel(st_g.r_vec, to_sm(st_s.r_vec, rperm)) < 1e-10
