"""Host-side logic of the drop-in (partition, config validation, scheduling, traces, inputs)."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as orc
from paper_1812_01307_b200 import blockops, problems, solvers, tv


def test_make_partition_matches_reference_golden():
    z = load_golden("partitions")
    k = 0
    while f"case{k}" in z:
        r, c, m, n = (int(v) for v in z[f"case{k}"])
        p = blockops.make_partition(r, c, m, n)
        assert np.array_equal(p.row_edges(), z[f"rows{k}"])
        assert np.array_equal(p.col_edges(), z[f"cols{k}"])
        assert p.num_row_blocks == m and p.num_col_blocks == n and p.rows == r and p.cols == c
        k += 1
    k = 0
    while f"err{k}" in z:
        with pytest.raises(ValueError):
            blockops.make_partition(*(int(v) for v in z[f"err{k}"]))
        k += 1


def test_spec_partition_example():
    p = blockops.make_partition(10, 8, 4, 4)
    assert p.row_sizes() == (3, 3, 2, 2) and p.col_sizes() == (2, 2, 2, 2)
    assert p.row_slice(1) == slice(3, 6) and p.col_range(3) == (6, 8)


@pytest.mark.parametrize("bounds,msg", [((), "empty"), (((1, 2),), "start at 0"),
                                        (((0, 2), (3, 4)), "contiguous"), (((0, 0),), "nonempty")])
def test_block_partition_validation(bounds, msg):
    with pytest.raises(ValueError, match=msg):
        blockops.BlockPartition(bounds, ((0, 1),))


@pytest.mark.parametrize("kw", [dict(mu=0), dict(mu=1, lam=-1), dict(mu=1, alpha=0), dict(mu=1, gamma=1.5),
                                dict(mu=1, epochs=-1), dict(mu=1, cg_iters=0), dict(mu=1, max_halvings=-1),
                                dict(mu=1, divergence_limit=0)])
def test_solver_config_validation(kw):
    with pytest.raises(ValueError):
        solvers.SolverConfig(**kw)


def test_prox_settings_validation():
    with pytest.raises(ValueError):
        tv.ProxSettings(0, 1e-5)
    with pytest.raises(ValueError):
        tv.ProxSettings(5, 0.0)


@pytest.mark.parametrize("m,n,a,g", [(4, 4, 1.0, 1.0), (8, 8, 1.0, 1.0), (4, 4, 0.5, 0.5), (3, 5, 0.4, 0.7)])
def test_schedule_pairs_advances_rng_like_the_reference(m, n, a, g):
    r1, r2 = np.random.default_rng(11), np.random.default_rng(11)
    for _ in range(5):
        assert solvers.schedule_pairs(m, n, a, g, r1) == orc.schedule_pairs(m, n, a, g, r2)
    assert r1.integers(1 << 30) == r2.integers(1 << 30)


def test_full_sweep_schedule_covers_every_pair_once():
    pairs = solvers.schedule_pairs(4, 4, 1.0, 1.0, np.random.default_rng(0))
    assert sorted(pairs) == [(i, j) for i in range(4) for j in range(4)]


def test_schedule_rejects_empty_selection():
    with pytest.raises(ValueError):
        solvers.schedule_pairs(2, 2, 0.1, 0.1, np.random.default_rng(0))


def test_trace_csv_roundtrip(tmp_path):
    tr = solvers.ConvergenceTrace()
    tr.append(solvers.TraceSample(0.0, 1.0, 12.5, 0.0))
    tr.append(solvers.TraceSample(1.0, 0.5, 3.25, 3.0))
    with pytest.raises(ValueError):
        tr.append(solvers.TraceSample(1.0, 0.4, 3.0, 4.0))
    p = tmp_path / "t.csv"
    tr.write_csv(p)
    back = solvers.read_trace_csv(p)
    assert back.samples == tr.samples
    assert tr.to_csv_string().splitlines()[0] == "epoch,relative_error,objective,matvec_units"


def test_trace_csv_matches_reference_format():
    z = load_golden("p1_ct")
    ref_csv = bytes(z["csv"]).decode()
    tr = solvers.ConvergenceTrace()
    for row in z["samples"]:
        tr.append(solvers.TraceSample(*[float(v) for v in row]))
    assert tr.to_csv_string() == ref_csv


def test_pixel_layout_roundtrip_and_validation():
    perm = np.random.default_rng(3).permutation(12)
    lay = tv.PixelLayout(3, 4, perm)
    x = np.arange(12.0)
    img = lay.to_image(x)
    assert np.array_equal(lay.to_vector(img), x)
    assert not lay.is_identity and tv.PixelLayout.row_major(3, 4).is_identity
    with pytest.raises(ValueError):
        tv.PixelLayout(3, 4, np.zeros(12, dtype=int))
    with pytest.raises(ValueError):
        tv.ImageGrid(0, 3, np.zeros(0))


def test_generators_are_deterministic_and_canonical():
    d1 = problems.config(0, scale=0.25)
    d2 = problems.config(0, scale=0.25)
    assert (d1.matrix != d2.matrix).nnz == 0 and np.array_equal(d1.y, d2.y)
    a = d1.matrix
    assert a.has_sorted_indices and a.has_canonical_format
    assert (a.data > 0).all()
    ls = problems.config(1, scale=1e-3)
    assert ls.matrix.shape == (2000, 500)
    assert (np.diff(ls.matrix.indptr) == 32).all()
    for r in range(0, 2000, 97):
        row = ls.matrix.indices[ls.matrix.indptr[r]:ls.matrix.indptr[r + 1]]
        assert len(np.unique(row)) == 32
    assert np.allclose(ls.y, ls.matrix.astype(np.float64) @ ls.x_true)


def test_parallel_beam_chord_lengths():
    # a uniform unit image projects to each ray's chord length through the square
    n = 16
    a = problems.parallel_beam_matrix(n, 8, 23)
    sums = np.asarray(a.sum(axis=1)).ravel()
    offsets = np.arange(23) - 11.0
    for ang in range(8):
        th = math.pi * ang / 8
        for b, o in enumerate(offsets):
            # chord of line {p : p.(cos, sin) = o} through [-n/2, n/2]^2
            c, s = math.cos(th), math.sin(th)
            ts = []
            for (p0, d) in ((o * c, -s), (o * s, c)):
                if abs(d) < 1e-15:
                    continue
                ts += [(-n / 2 - p0) / d, (n / 2 - p0) / d]
            lo, hi = -1e30, 1e30
            for (p0, d) in ((o * c, -s), (o * s, c)):
                if abs(d) < 1e-15:
                    if not -n / 2 <= p0 <= n / 2:
                        lo, hi = 0, 0
                    continue
                t1, t2 = (-n / 2 - p0) / d, (n / 2 - p0) / d
                lo, hi = max(lo, min(t1, t2)), min(hi, max(t1, t2))
            chord = max(0.0, hi - lo)
            assert abs(sums[ang * 23 + b] - chord) < 1e-9


def test_canonical_csr_sums_float32_duplicates_in_float64():
    """BlockOperator's canonical form (blockops.py:124-126): duplicates are summed in
    float64 as the reference does; float32 input stays float32 only when every
    summed value round-trips exactly, and an explicit dtype is honoured."""
    from scipy import sparse
    from paper_1812_01307_b200.blockops import _canonical_csr
    # 0.1f + 0.2f is not exactly representable in float32
    a = sparse.csr_array((np.array([0.1, 0.2, 3.0], dtype=np.float32), np.array([1, 1, 0]), np.array([0, 2, 3])),
                         shape=(2, 2))
    ref = sparse.csr_array(a.copy(), dtype=np.float64)   # (sum_duplicates mutates shared index arrays)
    ref.sum_duplicates()
    ref.sort_indices()
    c = _canonical_csr(a)
    assert c.dtype == np.float64 and np.array_equal(c.toarray(), ref.toarray())
    # exact sums keep float32
    b = sparse.csr_array((np.array([0.5, 0.25, 3.0], dtype=np.float32), np.array([1, 1, 0]), np.array([0, 2, 3])),
                         shape=(2, 2))
    cb = _canonical_csr(b)
    assert cb.dtype == np.float32 and cb.toarray()[0, 1] == 0.75
    # canonical float32 input is kept as is; explicit dtype wins
    d = sparse.random(30, 20, density=0.3, format="csr", dtype=np.float32, random_state=1)
    assert _canonical_csr(d).dtype == np.float32
    assert _canonical_csr(d, np.float64).dtype == np.float64
    with pytest.raises(ValueError):
        _canonical_csr(d, np.int32)


def test_distributed_driver_rejects_unsupported_modes():
    """DistributedBSGD raises instead of silently running a different algorithm: the
    stochastic pair subsets (alpha / gamma < 1, solvers.py:186-195) need a row-slab
    shard with pair products (they and enforce_decrease are supported there,
    tests/test_parallel_gloo.py), not a slice shard or an unknown backend."""
    import types
    from paper_1812_01307_b200 import parallel
    from paper_1812_01307_b200.solvers import SolverConfig
    for shard in (types.SimpleNamespace(), types.SimpleNamespace(owns_slices=True, pair_products=None)):
        for kw in ({"alpha": 0.5}, {"gamma": 0.5}):
            with pytest.raises(ValueError):
                parallel.DistributedBSGD(shard, np.zeros(4), SolverConfig(mu=0.1, **kw))


def test_slab_program_is_pw_combine():
    """The postfix program bsgd_slab_decide runs reproduces pw_combine bit for bit."""
    from paper_1812_01307_b200 import parallel
    rng = np.random.default_rng(0)
    for nvox, world, halo in ((1 << 20, 8, 4096), (1 << 16, 3, 256), (5000, 2, 50), (1 << 18, 5, 512)):
        slabs = parallel.prox_slabs(nvox, world, halo)
        vals = rng.standard_normal((world, 3)) * 10 ** rng.uniform(-8, 8, (world, 3))
        want = parallel.pw_combine(nvox, slabs, vals)
        stack = []
        for op in parallel.slab_program(nvox, slabs):
            if op >= 0:
                stack.append(list(vals[op]))
            else:
                b, a = stack.pop(), stack.pop()
                stack.append([x + y for x, y in zip(a, b)])
        assert len(stack) == 1 and stack[0] == want
