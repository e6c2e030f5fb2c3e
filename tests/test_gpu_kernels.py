"""CUDA kernel parity: SpMV (K1/K2), block products, patterns, TV prox, reductions.

Checked against the reference's own golden vectors (tests/golden) and the CPU
oracle (oracle/) on the same seeded inputs.  Floating-point tolerances: the
kernels differ from scipy only in the summation order inside a row (parallel
float64 reduction, FMA), so products agree to ~1e-15 relative; we assert
1e-12.  The TV prox mirrors the reference's elementwise rounding exactly and
differs only in the order of its three global sums: outputs 1e-10, ProxInfo
counts exact.
"""

import numpy as np
import pytest
from scipy import sparse

from conftest import golden_csr, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

SOLVER_CASES = ["p1_ct", "p2_morton", "p3_ls", "p4_div", "p1_stoch"]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)


@pytest.fixture(scope="module")
def B(cuda_ok):
    from paper_1812_01307_b200 import blockops, metrics, spectral, tv
    return blockops, tv, metrics, spectral


def _op(B, z, dtype=None):
    blockops = B[0]
    a = golden_csr(z)
    m, n = (int(v) for v in z["mn"])
    return blockops.BlockOperator(a, blockops.make_partition(a.shape[0], a.shape[1], m, n), dtype=dtype)


@pytest.mark.parametrize("case", SOLVER_CASES)
def test_block_products_vs_reference(B, case):
    z = load_golden(case)
    op = _op(B, z)
    part = op.partition
    xv, rv = z["probe_x"], z["probe_r"]
    for i in range(op.num_row_blocks):
        for j in range(op.num_col_blocks):
            zz = op.block_matvec(i, j, xv[part.col_slice(j)])
            gg = op.block_matvec_transpose(i, j, rv[part.row_slice(i)])
            assert rel(zz, z[f"z_{i}_{j}"]) < 1e-12
            assert rel(gg, z[f"gh_{i}_{j}"]) < 1e-12
            assert op.block_nnz(i, j) == int(z[f"nnz_{i}_{j}"])
    assert rel(op.matvec(xv), z["matvec"]) < 1e-12
    assert rel(op.rmatvec(rv), z["rmatvec"]) < 1e-12
    assert op.matvec_units == pytest.approx(4.0, abs=0)


@pytest.mark.parametrize("case", ["p1_ct", "p3_ls", "p2_morton"])
def test_block_patterns_bit_exact(B, case):
    z = load_golden(case)
    op = _op(B, z)
    oop = orc.OracleOperator(golden_csr(z), *(int(v) for v in z["mn"]))
    for i in range(op.num_row_blocks):
        for j in range(op.num_col_blocks):
            got, ref = op.block(i, j), oop.block_csr(i, j)
            assert got.shape == ref.shape
            assert np.array_equal(got.indptr, ref.indptr)
            assert np.array_equal(got.indices, ref.indices)
            assert np.array_equal(got.data, ref.data)
    indptr, indices, values = op.transpose_pattern()
    at = sparse.csr_array(golden_csr(z).T)
    at.sort_indices()
    assert np.array_equal(indptr, at.indptr) and np.array_equal(indices, at.indices)
    assert np.array_equal(values, at.data)


def test_float32_values_match_float64_products(B):
    z = load_golden("p3_ls")  # values are float32-representable
    op32 = _op(B, z, dtype=np.float32)
    op64 = _op(B, z, dtype=np.float64)
    assert op32.value_dtype == np.float32
    x = z["probe_x"]
    assert rel(op32.matvec(x), op64.matvec(x)) < 1e-14
    assert rel(op32.rmatvec(z["probe_r"]), z["rmatvec"]) < 1e-12


def test_device_tensors_in_and_out(B):
    import torch
    z = load_golden("p1_ct")
    op = _op(B, z)
    xt = torch.tensor(z["probe_x"], device="cuda")
    out = op.matvec(xt)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert rel(out.cpu().numpy(), z["matvec"]) < 1e-12


def test_product_validation_errors(B):
    z = load_golden("p1_ct")
    op = _op(B, z)
    with pytest.raises(ValueError):
        op.block_matvec(0, 0, np.zeros(3))
    with pytest.raises(ValueError):
        op.matvec(np.zeros(5))
    with pytest.raises(ValueError):
        B[0].BlockOperator(sparse.csr_array((3, 3)))
    with pytest.raises(ValueError, match="partition covers"):
        B[0].BlockOperator(golden_csr(z), B[0].make_partition(5, 5, 1, 1))


def test_assemble_residual(B):
    blockops = B[0]
    rng = np.random.default_rng(0)
    y = rng.standard_normal(37)
    zc = rng.standard_normal((5, 37))
    assert np.array_equal(blockops.assemble_residual(y, zc), orc.assemble_residual(y, zc))
    assert np.array_equal(blockops.assemble_residual(y, np.zeros((3, 37))), y)
    assert np.array_equal(blockops.assemble_residual(y, y[None, :]), np.zeros(37))
    with pytest.raises(ValueError):
        blockops.assemble_residual(y, np.zeros((2, 36)))


def test_empty_rows_and_empty_blocks(B):
    blockops = B[0]
    # block-diagonal with empty rows: off-diagonal blocks have nnz 0
    d = sparse.block_diag([sparse.random(30, 20, 0.2, random_state=1), sparse.random(30, 20, 0.2, random_state=2)])
    a = sparse.csr_array(d)
    a = sparse.csr_array(a.multiply(np.arange(60)[:, None] % 7 != 0))  # force empty rows
    op = blockops.BlockOperator(a, blockops.make_partition(60, 40, 2, 2))
    oop = orc.OracleOperator(a, 2, 2)
    assert op.block_nnz(0, 1) == 0 and op.block_nnz(1, 0) == 0
    x = np.random.default_rng(1).standard_normal(40)
    w = np.random.default_rng(2).standard_normal(60)
    assert rel(op.matvec(x), oop.matvec(x)) < 1e-12
    assert rel(op.rmatvec(w), oop.rmatvec(w)) < 1e-12
    assert np.array_equal(op.block_matvec(0, 1, x[20:]), np.zeros(30))
    assert op.block(0, 1).nnz == 0


@pytest.mark.parametrize("scale", [0.05, 1.0])
def test_c1_geometry_products_vs_oracle(B, scale):
    from paper_1812_01307_b200 import problems
    d = problems.config(0, scale=scale)
    blockops = B[0]
    op = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, 4, 4))
    oop = orc.OracleOperator(d.matrix, 4, 4)
    x = d.x_true
    w = np.random.default_rng(5).standard_normal(d.shape[0])
    assert rel(op.matvec(x), oop.matvec(x)) < 1e-12
    assert rel(op.rmatvec(w), oop.rmatvec(w)) < 1e-12
    for (i, j) in [(0, 0), (1, 3), (3, 2)]:
        r0, r1 = op.partition.row_range(i)
        c0, c1 = op.partition.col_range(j)
        assert rel(op.block_matvec(i, j, x[c0:c1]), oop.block_matvec(i, j, x[c0:c1])) < 1e-12
        assert rel(op.block_matvec_transpose(i, j, w[r0:r1]), oop.block_matvec_transpose(i, j, w[r0:r1])) < 1e-12


def test_c2_full_size_adjoint_and_linearity(B):
    """Full configs[1] size (2e6 x 5e5, 6.4e7 nnz): size-independent properties."""
    from paper_1812_01307_b200 import problems
    blockops = B[0]
    a = problems.random_sparse_system(2_000_000, 500_000, 32, 2)
    op = blockops.BlockOperator(a, blockops.make_partition(*a.shape, 8, 8))
    rng = np.random.default_rng(9)
    x, x2 = rng.standard_normal(500_000), rng.standard_normal(500_000)
    w = rng.standard_normal(2_000_000)
    ax, atw = op.matvec(x), op.rmatvec(w)
    assert abs(ax @ w - x @ atw) <= 1e-12 * np.linalg.norm(ax) * np.linalg.norm(w)
    lin = op.matvec(2.5 * x - x2)
    assert rel(lin, 2.5 * ax - op.matvec(x2)) < 1e-13
    # spot-check sampled blocks against the oracle restatement
    oop = orc.OracleOperator(a, 8, 8, threads=8)
    for (i, j) in [(0, 0), (7, 3)]:
        c0, c1 = op.partition.col_range(j)
        assert rel(op.block_matvec(i, j, x[c0:c1]), oop.block_matvec(i, j, x[c0:c1])) < 1e-12


# --- TV -------------------------------------------------------------------------

def test_tv_prox_vs_reference_golden(B):
    tv = B[1]
    z = load_golden("prox")
    for k in range(int(z["count"])):
        w, mi, tol = z[f"par{k}"]
        out, info = tv.tv_prox(tv.ImageGrid.from_matrix(z[f"in{k}"]), float(w),
                               tv.ProxSettings(int(mi), float(tol)), return_info=True)
        ref = z[f"out{k}"]
        assert rel(out.as_matrix(), ref) < 1e-10, k
        # numpy-order sums (csrc/pairwise.cuh): ProxInfo and dual values are bit-exact
        assert [info.iterations, int(info.converged), info.restarts, int(info.fell_back)] == list(z[f"info{k}"]), k
        if float(w) > 0:
            assert np.array_equal(np.array(info.dual_objectives), z[f"dual{k}"]), k
        assert np.array_equal(out.as_matrix(), ref), k
        assert tv.tv_value(out) == float(z[f"tv{k}"][1])
        assert tv.tv_value(tv.ImageGrid.from_matrix(z[f"in{k}"])) == float(z[f"tv{k}"][0])


def test_tv_prox_rows_kernel_vs_reference_golden(B):
    """Power-of-two images >= 128 wide run the row-walk kernel (csrc/fgp2.cu): output,
    ProxInfo and dual objectives bit-exact with the reference (restarts included)."""
    from golden_inputs import prox_rows_inputs
    tv = B[1]
    z = load_golden("prox_rows")
    for k, (name, img, w, mi, tol) in enumerate(prox_rows_inputs()):
        out, info = tv.tv_prox(tv.ImageGrid.from_matrix(img), w, tv.ProxSettings(mi, tol), return_info=True)
        assert np.array_equal(out.as_matrix(), z[f"out{k}"]), name
        assert [info.iterations, int(info.converged), info.restarts, int(info.fell_back)] == list(z[f"info{k}"]), name
        assert np.array_equal(np.array(info.dual_objectives), z[f"dual{k}"]), name
        assert tv.tv_value(out) == float(z[f"tv{k}"][1])


@pytest.mark.parametrize("shape,w,tol", [((1024, 1024), 0.01, 1e-300), ((1024, 1024), 2.0, 1e-300),
                                         ((512, 512), 0.05, 1e-12), ((128, 1024), 0.3, 1e-300),
                                         ((2048, 256), 0.02, 1e-9), ((256, 512), 1e-4, 1e-5)])
def test_tv_prox_rows_kernel_matches_cooperative_kernel(B, monkeypatch, shape, w, tol):
    """The row-walk kernel and the cooperative fgp_kernel<2> (BSGD_PROX_KERNEL=coop)
    give the same bits: output, ProxInfo, dual objectives, in standalone mode."""
    import torch
    tv = B[1]
    g = torch.Generator(device="cuda").manual_seed(sum(shape))
    img = torch.rand(*shape, dtype=torch.float64, device="cuda", generator=g) * 3.0
    img[shape[0] // 3:, : shape[1] // 2] += 1.0
    st = tv.ProxSettings(20, tol)
    outs = []
    for kernel in ("rows", "coop"):
        if kernel == "coop":
            monkeypatch.setenv("BSGD_PROX_KERNEL", "coop")
        out, info = tv.tv_prox(img, w, st, return_info=True)
        outs.append((out.cpu().numpy(), (info.iterations, info.converged, info.restarts, info.fell_back),
                     list(info.dual_objectives)))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1] and outs[0][2] == outs[1][2]


@pytest.mark.parametrize("shape,w", [((64, 64), 1e-3), ((64, 64), 0.05), ((37, 101), 0.2), ((200, 3), 1.0),
                                     ((256, 256), 0.01), ((1024, 1024), 0.01), ((1000, 999), 0.02)])
def test_tv_prox_vs_oracle_random(B, shape, w):
    tv = B[1]
    img = np.random.default_rng(sum(shape)).random(shape) * 2.0
    out, info = tv.tv_prox(tv.ImageGrid.from_matrix(img), w, tv.ProxSettings(20, 1e-12), return_info=True)
    ref, rep = orc.tv_prox(img, w, 20, 1e-12)
    assert np.array_equal(out.as_matrix(), ref)
    assert (info.iterations, info.restarts, info.fell_back) == (rep.iterations, rep.restarts, rep.fell_back)


def test_tv_prox_edge_cases(B):
    tv = B[1]
    img = tv.ImageGrid.from_matrix(np.random.default_rng(0).random((5, 6)))
    same, info = tv.tv_prox(img, 0.0, return_info=True)
    assert np.array_equal(same.data, img.data) and info.converged and info.iterations == 0
    const = tv.ImageGrid.from_matrix(np.full((7, 7), 5.0))
    assert np.array_equal(tv.tv_prox(const, 0.7).data, const.data)
    with pytest.raises(ValueError):
        tv.tv_prox(img, -1.0)
    one = tv.ImageGrid.from_matrix(np.array([[3.0]]))
    assert np.array_equal(tv.tv_prox(one, 1.0).data, one.data)


def test_tv_value_and_difference_operators(B):
    tv = B[1]
    z = load_golden("prox")
    assert tv.tv_value(tv.ImageGrid.from_matrix(np.array([[0.0, 1.0], [1.0, 1.0]]))) == float(z["tv_2x2"])
    assert tv.tv_value(tv.ImageGrid.from_matrix(np.array([[0.0, 3.0]]))) == 3.0
    assert tv.tv_value(tv.ImageGrid.from_matrix(np.full((4, 5), 2.0))) == 0.0
    gv, gh = tv.discrete_gradient(tv.ImageGrid.from_matrix(z["adj_u"]))
    assert np.array_equal(gv, z["adj_gv"]) and np.array_equal(gh, z["adj_gh"])
    dv = tv.discrete_divergence(z["adj_pv"], z["adj_ph"]).as_matrix()
    assert np.array_equal(dv, z["adj_div"])
    u = np.random.default_rng(4).random((9, 11))
    a = 3.7
    assert tv.tv_value(tv.ImageGrid.from_matrix(a * u)) == pytest.approx(a * tv.tv_value(tv.ImageGrid.from_matrix(u)),
                                                                         rel=1e-12)


def test_metrics_and_spectral(B):
    blockops, tv, metrics, spectral = B
    z = load_golden("p1_ct")
    op = _op(B, z)
    e = load_golden("p1_eig")
    res = spectral.largest_eigenvalue(op, max_iters=50)
    assert res.iterations == int(e["iterations"]) and res.converged == bool(int(e["converged"]))
    assert res.value == pytest.approx(float(e["value"]), rel=1e-10)
    x = z["final_x"]
    oop = orc.OracleOperator(golden_csr(z), 4, 5)
    assert metrics.relative_error(x, z["x_true"]) == pytest.approx(orc.relative_error(x, z["x_true"]), rel=1e-12)
    lay = tv.PixelLayout.row_major(24, 24)
    got = metrics.objective_value(x, op, z["y"], 5.0, lay)
    assert got == pytest.approx(orc.objective_value(x, oop, z["y"], 5.0, lay.perm, (24, 24)), rel=1e-12)
    with pytest.raises(ValueError):
        metrics.relative_error(x, np.zeros_like(x))
    sb = spectral.step_bound(9.0)
    assert sb.mu_sup == 1.0 / 18 and sb.admits(0.05) and not sb.admits(1 / 18)
    v1, v2 = spectral.iteration_eigenvalues(1.0, 0.5)
    assert abs(abs(v1) - 1.0) < 1e-12 and abs(abs(v2) - 1.0) < 1e-12


def test_gather_tiles_match_csr(B):
    """Gather-tiled products (gtile.cuh; kept whenever requested, no timing race)
    agree with the CSR kernel and the oracle to rounding; irregular tiles and
    removal work, and kernel_info reports which kernel runs."""
    blockops = B[0]
    from paper_1812_01307_b200 import problems
    n, ang, nb = 24, 20, 35
    a = problems.parallel_beam_matrix(n, ang, nb, dtype=np.float32)
    op = blockops.BlockOperator(a, blockops.make_partition(*a.shape, 4, 4))
    oop = orc.OracleOperator(a, 4, 4)
    rng = np.random.default_rng(3)
    x, w, y = rng.standard_normal(a.shape[1]), rng.standard_normal(a.shape[0]), rng.standard_normal(a.shape[0])
    op.set_gather_tiles(True, blockops.grid_tiles(n, n))
    perm = rng.permutation(a.shape[0])
    sizes = np.minimum(16, rng.integers(1, 17, size=a.shape[0]))
    ptr = np.concatenate([[0], np.cumsum(sizes)])
    ptr = ptr[ptr < a.shape[0]].tolist() + [a.shape[0]]
    op.set_gather_tiles(False, (np.asarray(ptr, dtype=np.int64), perm.astype(np.int64)))
    ki = op.kernel_info()
    assert ki["forward"] == "gather_tiled" and ki["transposed"] == "gather_tiled"
    assert rel(op.matvec(x), oop.matvec(x)) < 1e-12
    assert rel(op.rmatvec(w), oop.rmatvec(w)) < 1e-12
    r, s = op.residual_sumsq(x, y)
    want = y - oop.matvec(x)
    assert rel(r.cpu().numpy(), want) < 1e-12
    op.set_gather_tiles(True, None)
    op.set_gather_tiles(False, None)
    assert op.kernel_info()["transposed"] == "csr"
    assert rel(op.matvec(x), oop.matvec(x)) < 1e-12
    with pytest.raises(ValueError):
        op.set_gather_tiles(True, (np.array([0, 17]), np.arange(17)))


@pytest.mark.parametrize("dtype,lanes,compress", [(np.float32, "32", None), (np.float64, "32", "off"),
                                                  (np.float32, None, None), (np.float32, None, "off"),
                                                  (np.float64, "4", None), (np.float32, "4", "force"),
                                                  (np.float32, "16", "force")])
def test_blocked_stream_bit_identical(B, monkeypatch, dtype, lanes, compress):
    """The blocked copy of A's stream (spmv.cuh csr_blocked_kernel): with 32 lanes
    per row it gives the unblocked G = 32 kernel's products bit for bit (same
    per-lane order; padding adds exact zeros); with fewer lanes (the plan's
    choice, several rays per warp) it agrees to rounding.  Both index forms --
    plain int32 and the compressed 16-bit offsets from two bases per block (the
    structural rule keeps it at >= 8 lanes per ray; BSGD_BLK_COMPRESS forces either) --
    against the oracle, with kernel_info confirming which one ran.  Rows
    shorter than a block and empty rows included."""
    blockops = B[0]
    from paper_1812_01307_b200 import problems
    a = problems.parallel_beam_matrix(256, 24, 363, dtype=dtype)   # rays of up to ~360 nonzeros
    a = a.tolil()
    a[3, :] = 0          # an empty row
    a = a.tocsr()
    a.eliminate_zeros()
    part = blockops.make_partition(*a.shape, 2, 2)
    monkeypatch.setenv("BSGD_G_FWD", "32")     # the unblocked reference kernel: a warp per row
    monkeypatch.setenv("BSGD_NO_BLOCKED", "1")
    plain = blockops.BlockOperator(a, part)
    monkeypatch.delenv("BSGD_NO_BLOCKED")
    monkeypatch.setenv("BSGD_BLOCKED", "force")
    if lanes is not None:
        monkeypatch.setenv("BSGD_BLK_G", lanes)
    if compress is not None:
        monkeypatch.setenv("BSGD_BLK_COMPRESS", compress)
    blk = blockops.BlockOperator(a, part)
    g = int(lanes) if lanes is not None else 16    # tile-ordered gathers: 16 lanes per ray
    want_cmp = compress == "force" or (compress is None and g >= 8)
    ki = blk.kernel_info()
    assert ki["forward"] == ("blocked_compressed" if want_cmp else "blocked") and ki["forward_lanes"] == g
    assert ki["forward_order"] == "tile4"      # 256 x 256 image: gathers in 4 x 4 pixel tiles
    assert plain.kernel_info()["forward"] == "csr" and plain.kernel_info()["forward_lanes"] == 32
    exact = lanes == "32"
    oop = orc.OracleOperator(a, 2, 2)
    rng = np.random.default_rng(11)
    for _ in range(3):
        x = rng.standard_normal(a.shape[1])
        got = blk.matvec(x, charge=False)
        if exact:
            assert np.array_equal(got, plain.matvec(x, charge=False))
        assert rel(got, oop.matvec(x)) < 1e-12
        y = rng.standard_normal(a.shape[0])
        r1, s1 = blk.residual_sumsq(x, y)
        r0, s0 = plain.residual_sumsq(x, y)
        if exact:
            assert np.array_equal(r1.cpu().numpy(), r0.cpu().numpy())
        assert rel(r1.cpu().numpy(), y - oop.matvec(x)) < 1e-12


@pytest.mark.parametrize("lanes,compress", [(None, None), ("4", None), ("4", "force"), ("16", "off")])
def test_blocked_gather_order_bit_identical(B, monkeypatch, lanes, compress):
    """K1's tiled gather order (4 x 4 pixel tiles of a square image, the vector
    permuted the same way before the launch) keeps every entry at its position in
    the stream: products and residuals equal A's native column order bit for bit,
    with plain and compressed (16-bit offset) indices."""
    blockops = B[0]
    from paper_1812_01307_b200 import problems
    a = problems.parallel_beam_matrix(128, 30, 181, dtype=np.float32)
    part = blockops.make_partition(*a.shape, 2, 3)
    monkeypatch.setenv("BSGD_BLOCKED", "force")
    if lanes is not None:
        monkeypatch.setenv("BSGD_BLK_G", lanes)
    if compress is not None:
        monkeypatch.setenv("BSGD_BLK_COMPRESS", compress)
    tiled = blockops.BlockOperator(a, part)
    monkeypatch.setenv("BSGD_BLK_ORDER", "native")
    monkeypatch.setenv("BSGD_BLK_G", str(tiled.kernel_info()["forward_lanes"]))   # the order alone differs
    native = blockops.BlockOperator(a, part)
    kt, kn = tiled.kernel_info(), native.kernel_info()
    assert kt["forward_order"] == "tile4" and kn["forward_order"] == "native"
    assert kt["forward"] == kn["forward"] and kt["forward_lanes"] == kn["forward_lanes"]
    oop = orc.OracleOperator(a, 2, 3)
    rng = np.random.default_rng(4)
    for _ in range(3):
        x, y = rng.standard_normal(a.shape[1]), rng.standard_normal(a.shape[0])
        got = tiled.matvec(x, charge=False)
        assert np.array_equal(got, native.matvec(x, charge=False))
        assert rel(got, oop.matvec(x)) < 1e-12
        r1, s1 = tiled.residual_sumsq(x, y)
        r0, s0 = native.residual_sumsq(x, y)
        assert np.array_equal(r1.cpu().numpy(), r0.cpu().numpy()) and float(s1) == float(s0)


@pytest.mark.parametrize("grid,dtype", [("sinogram", np.float32), ("none", np.float32), ("sinogram", np.float64),
                                        ("sinogram4x4", np.float32), ("sinogram8x2", np.float32)])
def test_transposed_blocked_stream(B, monkeypatch, grid, dtype):
    """The blocked stream of A^T (bsgd_plan_blocked_transposed): 16 lanes per pixel
    row, gathers from r in sinogram tiles (the shape the plan picks from the gather
    footprint, and 4 x 4 / 8 x 2 forced; ragged last tiles: 30 angles, 181 bins) with
    16-bit offset indices, or in A^T's own order.  Lane l sums the entries = l mod 16
    in order and the lanes fold in the same shuffle tree as the gather-tiled kernel,
    so the two agree bit for bit; both against the oracle, through rmatvec and the
    epoch's step epilogue."""
    blockops, tv = B[0], B[1]
    from paper_1812_01307_b200 import problems, solvers
    n, ang, nb = 128, 30, 181
    a = problems.parallel_beam_matrix(n, ang, nb, dtype=dtype)
    part = blockops.make_partition(*a.shape, 2, 3)
    tiled = blockops.BlockOperator(a, part)
    tiled.set_gather_tiles(True, blockops.grid_tiles(n, n))
    blk = blockops.BlockOperator(a, part)
    if grid == "none":
        monkeypatch.setenv("BSGD_BLK_G_TR", "16")
    forced = {"sinogram4x4": ("1", "tile4"), "sinogram8x2": ("4", "tile8x2")}.get(grid)
    if forced:
        monkeypatch.setenv("BSGD_BLK_TILE", forced[0])
    blk.set_transposed_blocked(() if grid == "none" else (ang, nb))
    monkeypatch.delenv("BSGD_BLK_TILE", raising=False)
    ki = blk.kernel_info()
    assert ki["transposed"] == "blocked_compressed" and ki["transposed_lanes"] == 16
    # the plan picks the tile shape from the gather footprint (here, with only 30 angles,
    # the bins drift faster than the angles advance); the forced shapes cover the others
    if forced:
        assert ki["transposed_order"] == forced[1]
    else:
        assert ki["transposed_order"].startswith("tile") if grid == "sinogram" else ki["transposed_order"] == "native"
    assert tiled.kernel_info()["transposed"] == "gather_tiled"
    oop = orc.OracleOperator(a, 2, 3)
    rng = np.random.default_rng(8)
    for _ in range(3):
        w = rng.standard_normal(a.shape[0])
        got = blk.rmatvec(w, charge=False)
        assert np.array_equal(got, tiled.rmatvec(w, charge=False))
        assert rel(got, oop.rmatvec(w)) < 1e-12
    with pytest.raises(ValueError):
        blk.set_transposed_blocked((ang, nb + 1))
    # three TV epochs: the step epilogue on the blocked kernel
    d = rng.standard_normal(a.shape[0])
    cfg = solvers.SolverConfig(mu=1e-4, lam=0.5, epochs=3, prox=tv.ProxSettings(10, 1e-5))
    lay = tv.PixelLayout.row_major(n, n)
    s1, s2 = solvers.init_bsgd_state(blk, d, cfg), solvers.init_bsgd_state(tiled, d, cfg)
    for _ in range(3):
        solvers.bsgd_tv_iteration(s1, blk, d, cfg, layout=lay)
        solvers.bsgd_tv_iteration(s2, tiled, d, cfg, layout=lay)
    assert np.array_equal(s1.x, s2.x)
    blk.set_transposed_blocked(None)
    assert blk.kernel_info()["transposed"] == "csr"
    stacked = blockops.BlockOperator.stacked(problems.parallel_beam_matrix(8, 6, 11), 2,
                                             blockops.make_partition(6 * 11 * 2, 64 * 2, 2, 2))
    with pytest.raises(ValueError):
        stacked.set_transposed_blocked((6, 11))


@pytest.mark.parametrize("infer", [True, False])
def test_plain_csr_ct_system_gets_blocked_streams(B, monkeypatch, infer):
    """A CT system handed over as a plain scipy CSR (the reference's own call,
    blockops.py:123-152; no grid hints): rays and pixel rows are both long, so the plan
    builds the blocked stream of A (square image: tile order) and, on its own, a blocked
    stream of A^T -- gathered in tiles of the sinogram grid it infers from the gaps
    between A^T's consecutive entries (angles x bins = 400 x 363 here), or, with the
    inference off, in A^T's own column order; products, residual and two TV epochs
    against the oracle; naming the grid afterwards gives the tile order either way."""
    blockops, tv = B[0], B[1]
    from paper_1812_01307_b200 import problems, solvers
    n, ang, nb = 256, 400, 363                 # ~510 nonzeros per pixel row, ~230 per ray
    a = problems.parallel_beam_matrix(n, ang, nb, dtype=np.float32)
    assert a.nnz / a.shape[1] >= 384
    if not infer:
        monkeypatch.setenv("BSGD_NO_GRID_INFER", "1")
    op = blockops.BlockOperator(a, blockops.make_partition(*a.shape, 4, 4))
    ki = op.kernel_info()
    assert ki["transposed"] == "blocked_compressed"
    if infer:
        assert ki["transposed_lanes"] == 16 and ki["transposed_order"].startswith("tile")
    else:
        assert ki["transposed_lanes"] == 8 and ki["transposed_order"] == "native"
    oop = orc.OracleOperator(a, 4, 4)
    rng = np.random.default_rng(17)
    x, w = rng.standard_normal(a.shape[1]), rng.standard_normal(a.shape[0])
    assert rel(op.rmatvec(w, charge=False), oop.rmatvec(w)) < 1e-12
    assert rel(op.matvec(x, charge=False), oop.matvec(x)) < 1e-12
    y = rng.standard_normal(a.shape[0])
    mu = 1e-5
    cfg = solvers.SolverConfig(mu=mu, lam=0.5, epochs=2, prox=tv.ProxSettings(10, 1e-5))
    lay = tv.PixelLayout.row_major(n, n)
    st = solvers.init_bsgd_state(op, y, cfg)
    prm = orc.Params(mu=mu, lam=0.5, epochs=2, max_inner_iters=10, tol=1e-5)
    ost = orc.init_state(oop, y, prm)
    for _ in range(2):
        solvers.bsgd_tv_iteration(st, op, y, cfg, layout=lay)
        orc.epoch(ost, oop, y, prm, lay.perm, (n, n))
    assert rel(st.x, ost.x) < 1e-9 and rel(st.r_vec, ost.r_vec) < 1e-9
    op.set_transposed_blocked((ang, nb))
    ki = op.kernel_info()
    assert ki["transposed_order"].startswith("tile") and ki["transposed_lanes"] == 16
    assert rel(op.rmatvec(w, charge=False), oop.rmatvec(w)) < 1e-12
    op.set_gather_tiles(True, blockops.grid_tiles(n, n))      # the latest explicit request wins
    assert op.kernel_info()["transposed"] == "gather_tiled"
    assert rel(op.rmatvec(w, charge=False), oop.rmatvec(w)) < 1e-12


def test_forward_grid_inferred_for_non_square_image(B, monkeypatch):
    """A 128 x 256 image (not a square column space): the plan reads the image width off
    the rays' index gaps and gathers K1 in tile order; the products equal those of the
    plan without the inference (A's own column order) bit for bit -- only the order of
    the gathers differs -- and the oracle to rounding."""
    blockops = B[0]
    from paper_1812_01307_b200 import problems
    full = problems.parallel_beam_matrix(256, 60, 363, dtype=np.float32)
    a = sparse.csr_array(full[:, : 128 * 256])
    a.sort_indices()
    part = blockops.make_partition(*a.shape, 3, 2)
    monkeypatch.setenv("BSGD_BLOCKED", "force")
    monkeypatch.setenv("BSGD_BLK_G", "16")
    tiled = blockops.BlockOperator(a, part)
    monkeypatch.setenv("BSGD_NO_GRID_INFER", "1")
    native = blockops.BlockOperator(a, part)
    kt, kn = tiled.kernel_info(), native.kernel_info()
    assert kt["forward_order"].startswith("tile") and kn["forward_order"] == "native"
    assert kt["forward"] == kn["forward"] and kt["forward_lanes"] == kn["forward_lanes"] == 16
    oop = orc.OracleOperator(a, 3, 2)
    rng = np.random.default_rng(31)
    for _ in range(2):
        x = rng.standard_normal(a.shape[1])
        got = tiled.matvec(x, charge=False)
        assert np.array_equal(got, native.matvec(x, charge=False))
        assert rel(got, oop.matvec(x)) < 1e-12


@pytest.mark.parametrize("index", [2, 3])
def test_ct_full_size_products_consistent(B, index):
    """configs[2] / configs[3] at full size (2.4e8 / 1.9e9 nonzeros, projector built on
    the GPU) through the kernels the epoch uses -- tile-ordered blocked streams with 16-bit
    offset indices for A and A^T (asserted via kernel_info) -- against size-independent
    properties: adjointness, and agreement with the block-restricted kernels (a
    different reduction) on sampled row / column blocks."""
    from paper_1812_01307_b200 import problems
    d = problems.config_device(index)
    op = d.op
    ki = op.kernel_info()
    assert ki["forward"] == "blocked_compressed" and ki["forward_order"] == "tile4" and ki["forward_lanes"] == 16
    assert ki["transposed"] == "blocked_compressed" and ki["transposed_order"] == "tile8x2"
    rows, cols = op.shape
    rng = np.random.default_rng(index)
    x, w = rng.random(cols), rng.standard_normal(rows)
    ax, atw = op.matvec(x, charge=False), op.rmatvec(w, charge=False)
    assert abs(ax @ w - x @ atw) <= 1e-11 * np.linalg.norm(ax) * np.linalg.norm(w)
    m, n = op.partition.num_row_blocks, op.partition.num_col_blocks
    for i in (0, m // 2, m - 1):
        r0, r1 = op.partition.row_range(i)
        acc = np.zeros(r1 - r0)
        for j in range(n):
            c0, c1 = op.partition.col_range(j)
            acc += op.block_matvec(i, j, x[c0:c1])
        assert rel(ax[r0:r1], acc) < 1e-12
    for j in (0, n - 1):
        c0, c1 = op.partition.col_range(j)
        acc = np.zeros(c1 - c0)
        for i in range(m):
            r0, r1 = op.partition.row_range(i)
            acc += op.block_matvec_transpose(i, j, w[r0:r1])
        assert rel(atw[c0:c1], acc) < 1e-12


def test_prox_workspace_per_stream_and_thread(B):
    """Concurrent proxes never share a workspace: the cache key holds the current
    stream and thread; the same stream reuses its workspace."""
    import threading
    import torch
    tv = B[1]
    dev = torch.device("cuda", 0)
    w0 = tv.prox_workspace(64, 64, dev)
    assert tv.prox_workspace(64, 64, dev) is w0
    s1 = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s1):
        w1 = tv.prox_workspace(64, 64, dev)
    assert w1 is not w0
    other = []
    th = threading.Thread(target=lambda: other.append(tv.prox_workspace(64, 64, dev)))
    th.start()
    th.join()
    assert other[0] is not w0
    # two proxes of the same image on two streams give the same bits
    img = torch.rand(64, 64, dtype=torch.float64, device=dev)
    outs = []
    for st in (torch.cuda.current_stream(dev), s1):
        with torch.cuda.stream(st):
            outs.append(tv.tv_prox(img, 0.1, tv.ProxSettings(20, 1e-9)).clone())
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
