"""The opt-in panel-tiled SpMV (csrc/tiled.cuh, BSGD_TILED=2 keeps it without
autotuning) against the oracle.  Not on the default path (the CSR kernel wins on
every configuration measured), kept correct here."""

import numpy as np
import pytest

from conftest import golden_csr, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def test_panel_tiled_products_vs_oracle(cuda_ok, monkeypatch):
    monkeypatch.setenv("BSGD_TILED", "2")
    from paper_1812_01307_b200 import blockops, problems
    a = problems.random_sparse_system(3000, 1200, 24, seed=5)
    op = blockops.BlockOperator(a, blockops.make_partition(*a.shape, 4, 4))
    oop = orc.OracleOperator(a, 4, 4)
    rng = np.random.default_rng(1)
    x, w = rng.standard_normal(a.shape[1]), rng.standard_normal(a.shape[0])
    assert rel(op.matvec(x), oop.matvec(x)) < 1e-12
    assert rel(op.rmatvec(w), oop.rmatvec(w)) < 1e-12
    z = load_golden("p3_ls")
    g = golden_csr(z)
    op2 = blockops.BlockOperator(g, blockops.make_partition(*g.shape, 2, 2))
    xv = z["probe_x"]
    assert rel(op2.matvec(xv), z["matvec"]) < 1e-12
