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
