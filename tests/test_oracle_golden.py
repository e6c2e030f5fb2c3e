"""Pin the CPU oracle against golden vectors produced by the reference itself.

Every comparison here is bit-exact (np.array_equal): the oracle restates the
reference's arithmetic order (see oracle/oracle.py and oracle/bsgd_oracle.c).
"""

import numpy as np
import pytest

from conftest import golden_cfg, golden_csr, load_golden
from oracle import oracle as orc

SOLVER_CASES = ["p1_ct", "p2_morton", "p3_ls", "p4_div", "p1_stoch"]


def test_partitions_match_reference():
    z = load_golden("partitions")
    k = 0
    while f"case{k}" in z:
        r, c, m, n = (int(v) for v in z[f"case{k}"])
        rb, cb = orc.partition_bounds(r, c, m, n)
        assert np.array_equal(rb, z[f"rows{k}"])
        assert np.array_equal(cb, z[f"cols{k}"])
        k += 1
    k = 0
    while f"err{k}" in z:
        with pytest.raises(ValueError):
            orc.partition_bounds(*(int(v) for v in z[f"err{k}"]))
        k += 1


def test_prox_bit_exact():
    z = load_golden("prox")
    for k in range(int(z["count"])):
        w, mi, tol = z[f"par{k}"]
        out, rep = orc.tv_prox(z[f"in{k}"], float(w), int(mi), float(tol))
        assert np.array_equal(out, z[f"out{k}"]), k
        info = [rep.iterations, int(rep.converged), rep.restarts, int(rep.fell_back)]
        assert info == list(z[f"info{k}"]), k
        assert np.array_equal(np.array(rep.dual_objectives), z[f"dual{k}"]), k
        assert orc.tv_value(z[f"in{k}"]) == z[f"tv{k}"][0]
        assert orc.tv_value(out) == z[f"tv{k}"][1]


def test_prox_rows_bit_exact():
    """Power-of-two images >= 128 wide (the row-walk CUDA kernel's shapes), against
    the reference's own outputs, ProxInfo and dual objectives."""
    from golden_inputs import prox_rows_inputs
    z = load_golden("prox_rows")
    for k, (name, img, w, mi, tol) in enumerate(prox_rows_inputs()):
        out, rep = orc.tv_prox(img, w, mi, tol)
        assert np.array_equal(out, z[f"out{k}"]), name
        assert [rep.iterations, int(rep.converged), rep.restarts, int(rep.fell_back)] == list(z[f"info{k}"]), name
        assert np.array_equal(np.array(rep.dual_objectives), z[f"dual{k}"]), name


def test_tv_hand_values_and_adjointness():
    z = load_golden("prox")
    # SPEC.md:131 quotes 2+sqrt(2) for ((0,1),(1,1)); the reference itself returns 2
    # (that hand value belongs to ((0,1),(1,0))).  We pin the reference.
    assert float(z["tv_2x2"]) == 2.0 == orc.tv_value(np.array([[0.0, 1.0], [1.0, 1.0]]))
    assert abs(orc.tv_value(np.array([[0.0, 1.0], [1.0, 0.0]])) - (2 + np.sqrt(2))) < 1e-12
    assert float(z["tv_1x2"]) == 3.0
    gv, gh = orc.forward_diff(z["adj_u"])
    assert np.array_equal(gv, z["adj_gv"]) and np.array_equal(gh, z["adj_gh"])
    dv = orc.divergence(z["adj_pv"], z["adj_ph"])
    assert np.array_equal(dv, z["adj_div"])
    lhs = np.sum(gv * z["adj_pv"]) + np.sum(gh * z["adj_ph"])
    rhs = -np.sum(z["adj_u"] * dv)
    assert abs(lhs - rhs) < 1e-12


def _operator(z):
    m, n = (int(v) for v in z["mn"])
    return orc.OracleOperator(golden_csr(z), m, n, threads=4)


@pytest.mark.parametrize("case", SOLVER_CASES)
def test_block_products_bit_exact(case):
    z = load_golden(case)
    op = _operator(z)
    xv, rv = z["probe_x"], z["probe_r"]
    for i in range(op.M):
        for j in range(op.N):
            r0, r1 = op.row_bounds[i], op.row_bounds[i + 1]
            c0, c1 = op.col_bounds[j], op.col_bounds[j + 1]
            assert np.array_equal(op.block_matvec(i, j, xv[c0:c1]), z[f"z_{i}_{j}"])
            assert np.array_equal(op.block_matvec_transpose(i, j, rv[r0:r1]), z[f"gh_{i}_{j}"])
            assert op.block_nnz(i, j) == int(z[f"nnz_{i}_{j}"])
    assert np.array_equal(op.matvec(xv), z["matvec"])
    assert np.array_equal(op.rmatvec(rv), z["rmatvec"])
    # every block charged twice (forward + transposed) plus two full products
    assert op.applied == 4 * op.nnz


def _params(cfg):
    return orc.Params(mu=cfg["mu"], lam=cfg["lam"], alpha=cfg["alpha"], gamma=cfg["gamma"],
                      epochs=cfg["epochs"], seed=cfg["seed"], max_inner_iters=cfg["max_inner_iters"],
                      tol=cfg["tol"], monitor_decrease=cfg["monitor_decrease"],
                      enforce_decrease=cfg["enforce_decrease"], max_halvings=cfg["max_halvings"],
                      divergence_limit=cfg["divergence_limit"])


def _layout(z):
    if "perm" in z:
        return z["perm"], tuple(int(v) for v in z["hw"])
    return None, None


@pytest.mark.parametrize("case", SOLVER_CASES)
def test_epochs_bit_exact(case):
    z = load_golden(case)
    op = _operator(z)
    prm = _params(golden_cfg(z))
    perm, hw = _layout(z)
    st = orc.init_state(op, z["y"], prm)
    for e in range(3):
        orc.epoch(st, op, z["y"], prm, perm, hw)
        assert np.array_equal(st.x, z[f"ep{e}_x"]), (case, e)
        assert np.array_equal(st.r_vec, z[f"ep{e}_r"]), (case, e)
        assert np.array_equal(st.g, z[f"ep{e}_g"]), (case, e)
        f, mu, ep, ok = z[f"ep{e}_scalars"]
        assert st.f_curr == f and st.mu_eff == mu and st.epoch == ep
        assert (-1 if st.last_decrease_ok is None else int(st.last_decrease_ok)) == ok


@pytest.mark.parametrize("case", SOLVER_CASES)
def test_run_bsgd_bit_exact(case):
    z = load_golden(case)
    op = _operator(z)
    cfg = golden_cfg(z)
    perm, hw = _layout(z)
    op.applied = int(z["applied0"])  # the reference ran on an operator with prior charges
    res = orc.run_bsgd(op, z["y"], _params(cfg), x_true=z["x_true"], perm=perm, hw=hw,
                       sample_every=cfg["sample_every"])
    samples = np.array(res.samples, dtype=np.float64).reshape(-1, 4)
    assert np.array_equal(samples, z["samples"]), case
    flags = [int(f) for f in res.decrease_flags]
    assert flags == list(z["flags"])
    assert res.diverged == bool(int(z["diverged"]))
    if res.diverged:
        assert res.message == bytes(z["message"]).decode().split(": ", 1)[-1] or \
            res.message in bytes(z["message"]).decode()
    else:
        assert np.array_equal(res.final_x, z["final_x"])


@pytest.mark.parametrize("case,eig", [("p1_ct", "p1_eig"), ("p3_ls", "p3_eig")])
def test_largest_eigenvalue_bit_exact(case, eig):
    z = load_golden(case)
    e = load_golden(eig)
    op = orc.OracleOperator(golden_csr(z), 4 if case == "p1_ct" else 8, 5 if case == "p1_ct" else 8)
    val, conv, its = orc.largest_eigenvalue(op, max_iters=50)
    assert val == float(e["value"]) and int(conv) == int(e["converged"]) and its == int(e["iterations"])


def _pairwise(a, lo, n):
    """numpy's pairwise_sum restated (the algorithm csrc/pairwise.cuh evaluates on the GPU)."""
    if n < 8:
        r = 0.0
        for i in range(lo, lo + n):
            r += a[i]
        return r
    if n <= 128:
        acc = [a[lo + j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                acc[j] += a[lo + i + j]
            i += 8
        res = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))
        while i < n:
            res += a[lo + i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(a, lo, n2) + _pairwise(a, lo + n2, n - n2)


@pytest.mark.parametrize("shape", [(5,), (17,), (128,), (129,), (24, 24), (37, 101), (200, 3), (256, 256),
                                   (300, 301), (4, 3, 5), (16, 16, 16), (5, 40, 7), (32, 32, 32)])
def test_numpy_pairwise_restatement(shape):
    """np.sum over a contiguous array == the pairwise recursion over its flat data, bit for bit."""
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape) * 10.0 ** rng.uniform(-3, 3, shape)
    assert float(np.sum(x)) == _pairwise(x.ravel().tolist(), 0, x.size)
    assert float(np.sum(x * x)) == _pairwise((x * x).ravel().tolist(), 0, x.size)


# --- 3-D extension (configs[4]); PARITY UNPINNED: no reference implementation ----

def test_oracle_3d_operators_are_adjoint():
    rng = np.random.default_rng(7)
    u = rng.standard_normal((5, 6, 7))
    p = [rng.standard_normal(u.shape) for _ in range(3)]
    g = orc.forward_diff3(u)
    lhs = sum(float(np.sum(a * b)) for a, b in zip(g, p))
    assert lhs == pytest.approx(-float(np.sum(u * orc.divergence3(*p))), rel=1e-12)
    # a volume constant along z has 3-D TV = sum over slices of the 2-D TV
    img = rng.random((9, 11))
    vol = np.repeat(img[None], 4, axis=0)
    assert orc.tv_value3(vol) == pytest.approx(4 * orc.tv_value(img), rel=1e-12)


def test_oracle_3d_prox_decreases_energy():
    rng = np.random.default_rng(8)
    b = rng.random((6, 8, 10))
    for w in (0.01, 0.1, 1.0):
        out, rep = orc.tv_prox3(b, w, 50, 1e-10)
        assert orc._prox_energy3(out, b, w) <= orc._prox_energy3(b, b, w)
        duals = rep.dual_objectives
        assert all(duals[k + 1] <= duals[k] for k in range(len(duals) - 1))


def test_oracle_3d_epoch_runs():
    """run_bsgd on a slice-stacked system uses the 3-D prox (hw of length 3)."""
    from scipy import sparse
    from paper_1812_01307_b200 import problems
    a2 = problems.parallel_beam_matrix(8, 6, 11)
    d = 3
    a = sparse.csr_array(sparse.kron(a2, sparse.identity(d), format="csr"))
    a.sort_indices()
    n = a2.shape[1]
    perm = np.array([z * n + p for p in range(n) for z in range(d)])
    op = orc.OracleOperator(a, 2, 2)
    x_true = np.random.default_rng(0).random(a.shape[1])
    y = a @ x_true
    eig, _, _ = orc.largest_eigenvalue(op)
    prm = orc.Params(mu=0.9 / (2 * eig), lam=0.01, epochs=3, max_inner_iters=5)
    res = orc.run_bsgd(op, y, prm, x_true=x_true, perm=perm, hw=(d, 8, 8))
    assert len(res.samples) == 4 and res.samples[-1][1] < res.samples[0][1]


def _tv3_independent(t):
    """Isotropic 3-D TV written from np.diff (shares no code with the oracle)."""
    g2 = np.zeros(t.shape)
    g2[1:, :, :] += np.diff(t, axis=0) ** 2
    g2[:, 1:, :] += np.diff(t, axis=1) ** 2
    g2[:, :, 1:] += np.diff(t, axis=2) ** 2
    return float(np.sqrt(g2).sum())


def test_oracle_3d_prox_reduces_to_reference_pinned_2d_prox():
    """A volume constant along z has a z-constant minimiser whose slices solve the 2-D
    problem, so tv_prox3 must reproduce the 2-D tv_prox (pinned bit-exact to the reference,
    tv.py:172-255) on every slice: ties the unpinned 3-D restatement to the pinned 2-D one."""
    rng = np.random.default_rng(21)
    img = rng.random((12, 15))
    img[3:8, 4:11] += 1.0
    vol = np.repeat(img[None], 5, axis=0)
    for w in (0.02, 0.3):
        ref2, rep2 = orc.tv_prox(img, w, 4000, 1e-12)
        out3, rep3 = orc.tv_prox3(vol, w, 4000, 1e-12)
        assert not rep2.fell_back and not rep3.fell_back
        assert np.abs(out3 - out3[:1]).max() < 1e-8          # z-constant
        assert np.abs(out3[2] - ref2).max() < 1e-7


def test_oracle_3d_prox_is_the_minimiser():
    """Optimality against an independent statement of the 3-D problem: the prox output's
    energy ||t - b||^2 + 2 w TV3(t) (TV from np.diff, not the oracle's operators) is not
    improved by an independent Chambolle-Pock solve nor by random perturbations."""
    rng = np.random.default_rng(22)
    b = rng.random((7, 9, 8))
    b[2:5, 3:7, 1:6] += 0.8
    w = 0.15
    out, rep = orc.tv_prox3(b, w, 3000, 1e-12)
    assert not rep.fell_back

    def energy(t):
        return float(((t - b) ** 2).sum()) + 2.0 * w * _tv3_independent(t)

    # Chambolle-Pock on min_t 0.5 ||t - b||^2 + w ||D t||_{2,1}, D from np.diff
    def grad(t):
        g = np.zeros((3,) + t.shape)
        g[0, 1:] = np.diff(t, axis=0)
        g[1, :, 1:] = np.diff(t, axis=1)
        g[2, :, :, 1:] = np.diff(t, axis=2)
        return g

    def grad_t(g):                    # adjoint of grad
        t = np.zeros(g.shape[1:])
        t[1:] += g[0, 1:]
        t[:-1] -= g[0, 1:]
        t[:, 1:] += g[1, :, 1:]
        t[:, :-1] -= g[1, :, 1:]
        t[:, :, 1:] += g[2, :, :, 1:]
        t[:, :, :-1] -= g[2, :, :, 1:]
        return t

    t = b.copy()
    tb = t.copy()
    dual = np.zeros((3,) + b.shape)
    sigma = tau = 1.0 / np.sqrt(12.0)
    for _ in range(6000):
        dual = dual + sigma * grad(tb)
        dual /= np.maximum(1.0, np.sqrt((dual ** 2).sum(axis=0)) / w)
        t_new = (t - tau * grad_t(dual) + tau * b) / (1.0 + tau)
        tb = 2.0 * t_new - t
        t = t_new
    assert np.linalg.norm(out - t) / np.linalg.norm(t) < 2e-5   # plain CP converges at O(1/k)
    e0 = energy(out)
    assert e0 <= energy(t) + 1e-9
    for _ in range(20):
        d = rng.standard_normal(b.shape)
        assert e0 <= energy(out + 1e-4 * d) and e0 <= energy(out - 1e-4 * d)
