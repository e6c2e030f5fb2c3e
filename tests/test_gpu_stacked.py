"""Slice-stacked operator (configs[4]) against the oracle on the expanded CSR.

`BlockOperator.stacked(A2, D)` stores only the 2-D slice matrix; the oracle
gets the full interleaved matrix kron(A2, I_D).  The stacked kernels follow the
reference's block-sequential arithmetic (one multiply and one add per term,
block segments folded in order), so every product is BIT-EXACT against the
oracle, and so is the x trajectory of a TV-regularised run (3-D prox included);
only the Eq. 9 monitor value and sampled objectives use a different reduction
order (1e-12 relative).
"""

import numpy as np
import pytest
from scipy import sparse

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M(cuda_ok):
    from paper_1812_01307_b200 import blockops, problems, solvers, spectral, tv
    return blockops, problems, solvers, spectral, tv


def _expanded(a2, depth):
    a = sparse.csr_array(sparse.kron(sparse.csr_array(a2), sparse.identity(depth, format="csr"), format="csr"))
    a.sort_indices()
    return a


CASES = [(8, 6, 11, 3, 2, 3, np.float64), (8, 6, 11, 16, 3, 2, np.float32), (6, 5, 9, 40, 4, 4, np.float64),
         (10, 8, 15, 64, 16, 16, np.float32), (5, 4, 7, 33, 1, 1, np.float64)]


@pytest.mark.parametrize("n,ang,nb,depth,m,nblk,dt", CASES)
def test_stacked_products_bit_exact(M, n, ang, nb, depth, m, nblk, dt):
    blockops, problems = M[0], M[1]
    a2 = problems.parallel_beam_matrix(n, ang, nb, dtype=dt)
    a = _expanded(a2, depth)
    part = blockops.make_partition(a.shape[0], a.shape[1], m, nblk)
    op = blockops.BlockOperator.stacked(a2, depth, part)
    oop = orc.OracleOperator(a, m, nblk)
    assert op.shape == a.shape and op.nnz == a.nnz and op.depth == depth
    rng = np.random.default_rng(depth)
    x = rng.standard_normal(a.shape[1])
    r = rng.standard_normal(a.shape[0])
    assert np.array_equal(op.matvec(x), oop.matvec(x))
    assert np.array_equal(op.rmatvec(r), oop.rmatvec(r))
    for i in range(m):
        for j in range(nblk):
            assert op.block_nnz(i, j) == oop.block_nnz(i, j)
            r0, r1 = part.row_range(i)
            c0, c1 = part.col_range(j)
            blk = oop.block_csr(i, j)
            got = op.block(i, j)
            assert np.array_equal(got.indptr, blk.indptr) and np.array_equal(got.indices, blk.indices)
            assert np.array_equal(got.data, blk.data)
            zs, gs = oop.pair_products([(i, j)], x, r)
            assert np.array_equal(op.block_matvec(i, j, x[c0:c1]), zs[0])
            assert np.array_equal(op.block_matvec_transpose(i, j, r[r0:r1]), gs[0])
    csr = op.tocsr()
    assert np.array_equal(csr.indptr, a.indptr) and np.array_equal(csr.indices, a.indices)
    assert np.array_equal(csr.data, a.data)
    ip, ix, vv = op.transpose_pattern()
    at = sparse.csr_array(a.T)
    at.sort_indices()
    assert np.array_equal(ip, at.indptr) and np.array_equal(ix, at.indices) and np.array_equal(vv, at.data)


def test_stacked_residual_and_errors(M):
    blockops, problems = M[0], M[1]
    a2 = problems.parallel_beam_matrix(8, 6, 11)
    depth = 5
    a = _expanded(a2, depth)
    op = blockops.BlockOperator.stacked(a2, depth, blockops.make_partition(*a.shape, 2, 2))
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(a.shape[1]), rng.standard_normal(a.shape[0])
    r, s = op.residual_sumsq(x, y)
    want = y - a @ x
    assert np.allclose(r.cpu().numpy(), want, rtol=0, atol=1e-12 * np.abs(want).max())
    assert float(s.item()) == pytest.approx(float(want @ want), rel=1e-12)
    with pytest.raises(ValueError):
        blockops.BlockOperator.stacked(a2, 1)
    with pytest.raises(ValueError):
        blockops.BlockOperator.stacked(a2, depth, blockops.make_partition(a.shape[0] + 1, a.shape[1], 1, 1))


@pytest.mark.parametrize("lam,alpha,epochs,view", [(0.01, 1.0, 6, "slice_major"), (0.0, 1.0, 5, "slice_major"),
                                                    (0.02, 0.5, 6, "slice_major"), (0.01, 1.0, 6, "native")])
def test_stacked_run_vs_oracle_bit_exact(M, lam, alpha, epochs, view):
    """TV-regularised (3-D prox) and least-squares runs: x bit-identical to the oracle."""
    blockops, problems, solvers, spectral, tv = M
    n, depth, m = 12, 8, 4
    a2 = problems.parallel_beam_matrix(n, 10, 17)
    a = _expanded(a2, depth)
    op = blockops.BlockOperator.stacked(a2, depth, blockops.make_partition(*a.shape, m, m))
    vol = problems.ellipsoid_phantom(n, depth, 6, 0)
    x_true = np.ascontiguousarray(vol.reshape(depth, n * n).T).ravel()
    y = a @ x_true + np.random.default_rng(1).standard_normal(a.shape[0]) * 0.01
    oop = orc.OracleOperator(a, m, m)
    u, _, _ = orc.largest_eigenvalue(oop)
    mu = 0.9 / (2.0 * u)
    if view == "slice_major":   # (slices, rows, cols) volume through the permutation
        perm = problems.interleaved_perm(n * n, depth)
        shape = (depth, n, n)
    else:                       # the interleaved vector is the (rows, cols, slices) volume
        perm = np.arange(n * n * depth)
        shape = (n, n, depth)
    layout = tv.VolumeLayout(*shape, perm) if lam > 0 else None
    cfg = solvers.SolverConfig(mu=mu, lam=lam, alpha=alpha, gamma=alpha, epochs=epochs, seed=3,
                               prox=tv.ProxSettings(10, 1e-5))
    tr = solvers.run_solver("bsgd", solvers.Problem(op, y, x_true, layout), cfg)
    prm = orc.Params(mu=mu, lam=lam, alpha=alpha, gamma=alpha, epochs=epochs, seed=3, max_inner_iters=10, tol=1e-5)
    ref = orc.run_bsgd(oop, y, prm, x_true=x_true, perm=perm if lam > 0 else None, hw=shape)
    assert np.array_equal(tr.final_x, ref.final_x)
    got = np.array([tuple(s) for s in tr.samples])
    want = np.array(ref.samples)
    assert np.array_equal(got[:, 0], want[:, 0])
    assert np.allclose(got[:, 1], want[:, 1], rtol=1e-12)
    assert np.allclose(got[:, 2], want[:, 2], rtol=1e-12)


def test_stacked_device_generator_matches_host(M):
    """from_parallel_beam(depth=D) == BlockOperator.stacked(parallel_beam_matrix(...), D)."""
    blockops, problems = M[0], M[1]
    n, ang, nb, depth = 16, 12, 23, 7
    dev = blockops.BlockOperator.from_parallel_beam(n, ang, nb, 2, 2, dtype=np.float32, depth=depth)
    a2 = problems.parallel_beam_matrix(n, ang, nb, dtype=np.float32)
    host = blockops.BlockOperator.stacked(a2, depth, blockops.make_partition(*dev.shape, 2, 2))
    assert dev.nnz == host.nnz
    x = np.random.default_rng(2).random(dev.shape[1])
    assert np.array_equal(dev.matvec(x), host.matvec(x))
    d = problems.config_device(4, scale=0.0625)
    assert d.op.depth == d.depth == 16 and d.op.shape[1] == 16 * 16 * 16
    assert d.layout().size == d.op.shape[1] and d.layout().is_identity
    assert d.layout(slice_major=True).size == d.op.shape[1]


@pytest.mark.parametrize("depth,m,dt", [(128, 4, np.float32), (256, 16, np.float32), (128, 3, np.float32),
                                        (128, 5, np.float64)])
def test_tile_staged_products_bit_exact(M, depth, m, dt):
    """Tile-staged stacked products (shared-memory windows over each tile's distinct
    columns) equal the untiled kernel and the oracle bit for bit."""
    blockops, problems = M[0], M[1]
    n, ang, nb = 12, 10, 17
    a2 = problems.parallel_beam_matrix(n, ang, nb, dtype=dt)
    a = _expanded(a2, depth)
    part = blockops.make_partition(a.shape[0], a.shape[1], m, m)
    plain = blockops.BlockOperator.stacked(a2, depth, part)
    tiled = blockops.BlockOperator.stacked(a2, depth, part)
    tiled.set_stacked_tiles(True, blockops.grid_tiles(n, n))
    tiled.set_stacked_tiles(False, blockops.grid_tiles(ang, nb, 4, 4))
    oop = orc.OracleOperator(a, m, m)
    rng = np.random.default_rng(depth)
    x = rng.standard_normal(a.shape[1])
    r = rng.standard_normal(a.shape[0])
    assert np.array_equal(tiled.matvec(x), oop.matvec(x))
    assert np.array_equal(tiled.rmatvec(r), oop.rmatvec(r))
    assert np.array_equal(tiled.matvec(x), plain.matvec(x))
    y = rng.standard_normal(a.shape[0])
    rt, st = tiled.residual_sumsq(x, y)
    rp, sp = plain.residual_sumsq(x, y)
    assert np.array_equal(rt.cpu().numpy(), rp.cpu().numpy())
    tiled.set_stacked_tiles(False, None)   # removable
    assert np.array_equal(tiled.matvec(x), oop.matvec(x))
    with pytest.raises(ValueError):
        tiled.set_stacked_tiles(True, (np.array([0, 3]), np.array([0, 1, 2])))   # must cover all rows


def test_tile_staged_run_bit_exact(M):
    """Device-generated stacked operator with tiles (the configs[4] path): run == oracle."""
    blockops, problems, solvers, spectral, tv = M
    n, depth, ang, nb = 8, 128, 6, 11
    op = blockops.BlockOperator.from_parallel_beam(n, ang, nb, 4, 4, dtype=np.float32, depth=depth, tiles=True)
    a2 = problems.parallel_beam_matrix(n, ang, nb, dtype=np.float32)
    a = _expanded(a2, depth)
    vol = problems.ellipsoid_phantom(n, depth, 6, 0)
    x_true = np.ascontiguousarray(vol.reshape(depth, n * n).T).ravel()
    y = a @ x_true + np.random.default_rng(1).standard_normal(a.shape[0]) * 0.01
    oop = orc.OracleOperator(a, 4, 4)
    u, _, _ = orc.largest_eigenvalue(oop)
    layout = tv.VolumeLayout.z_major(n, n, depth)
    cfg = solvers.SolverConfig(mu=0.9 / (2 * u), lam=0.01, epochs=5, seed=3, prox=tv.ProxSettings(10, 1e-5))
    tr = solvers.run_solver("bsgd", solvers.Problem(op, y, x_true, layout), cfg)
    prm = orc.Params(mu=cfg.mu, lam=0.01, epochs=5, seed=3, max_inner_iters=10, tol=1e-5)
    ref = orc.run_bsgd(oop, y, prm, x_true=x_true, perm=np.arange(a.shape[1]), hw=(n, n, depth))
    assert np.array_equal(tr.final_x, ref.final_x)


def test_tile_staged_irregular_tiles_and_empty_rows(M):
    """Random row groupings (tiles of 1..16 rows, any order), empty rows and columns,
    and a partition whose bounds are not multiples of D: still bit-exact."""
    blockops = M[0]
    rng = np.random.default_rng(11)
    r2, c2, depth = 90, 70, 128
    dense = (rng.random((r2, c2)) < 0.08) * rng.standard_normal((r2, c2))
    dense[[3, 17, 40], :] = 0.0          # empty rows
    dense[:, [0, 5, 66]] = 0.0           # empty columns
    a2 = sparse.csr_array(dense.astype(np.float32))
    a2.eliminate_zeros()
    a = _expanded(a2, depth)
    part = blockops.make_partition(a.shape[0], a.shape[1], 7, 5)
    op = blockops.BlockOperator.stacked(a2, depth, part)

    def random_tiles(n):
        perm = rng.permutation(n)
        sizes, tot = [], 0
        while tot < n:
            k = int(min(n - tot, rng.integers(1, 17)))
            sizes.append(k)
            tot += k
        return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64), perm.astype(np.int64)

    op.set_stacked_tiles(False, random_tiles(r2))
    op.set_stacked_tiles(True, random_tiles(c2))
    oop = orc.OracleOperator(a, 7, 5)
    x = rng.standard_normal(a.shape[1])
    r = rng.standard_normal(a.shape[0])
    assert np.array_equal(op.matvec(x), oop.matvec(x))
    assert np.array_equal(op.rmatvec(r), oop.rmatvec(r))


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


def test_configs4_full_size_adjoint(M):
    """configs[4] at full size (256^3, 7.7e9 logical nonzeros) through the tile-staged
    products: adjointness and agreement of a sampled block pair with the
    block-restricted stacked kernel."""
    from paper_1812_01307_b200 import problems
    d = problems.config_device(4)
    op = d.op
    rows, cols = op.shape
    rng = np.random.default_rng(4)
    x, w = rng.random(cols), rng.standard_normal(rows)
    ax, atw = op.matvec(x, charge=False), op.rmatvec(w, charge=False)
    assert abs(ax @ w - x @ atw) <= 1e-11 * np.linalg.norm(ax) * np.linalg.norm(w)
    m, n = op.partition.num_row_blocks, op.partition.num_col_blocks
    i = m // 2                      # interleaved order: every (i, j) block holds entries
    r0, r1 = op.partition.row_range(i)
    parts = [op.block_matvec(i, j, x[slice(*op.partition.col_range(j))]) for j in range(n)]
    # the tile kernel folds the block segments as r = ((0 + s_0) + s_1) + ...
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = acc + p
    assert _rel(acc, ax[r0:r1]) < 1e-13
    j = n - 1
    c0, c1 = op.partition.col_range(j)
    parts = [op.block_matvec_transpose(k, j, w[slice(*op.partition.row_range(k))]) for k in range(m)]
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = acc + p
    assert _rel(acc, atw[c0:c1]) < 1e-13
