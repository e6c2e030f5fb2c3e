"""Device Siddon generator against the host generator and geometry."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,ang,bins,dtype", [(16, 8, 23, np.float64), (24, 30, 35, np.float32),
                                              (128, 180, 183, np.float64), (64, 37, 91, np.float32),
                                              (33, 20, 47, np.float64)])
def test_device_matrix_bit_identical_to_host(cuda_ok, n, ang, bins, dtype):
    from paper_1812_01307_b200 import blockops, problems
    host = problems.parallel_beam_matrix(n, ang, bins, dtype=dtype)
    op = blockops.BlockOperator.from_parallel_beam(n, ang, bins, 2, 3, dtype=dtype)
    dev = op.tocsr()
    assert dev.shape == host.shape and dev.nnz == host.nnz
    assert np.array_equal(dev.indptr, host.indptr)
    assert np.array_equal(dev.indices, host.indices)
    assert dev.data.dtype == host.data.dtype and np.array_equal(dev.data, host.data)
    ref = blockops.BlockOperator(host, blockops.make_partition(*host.shape, 2, 3))
    assert [[op.block_nnz(i, j) for j in range(3)] for i in range(2)] == \
           [[ref.block_nnz(i, j) for j in range(3)] for i in range(2)]


def test_configs3_size_generation_and_chords(cuda_ok):
    """configs[3] geometry (1024^2, 1440 x 1449): a uniform image projects to chord lengths."""
    from paper_1812_01307_b200 import blockops
    n, ang, bins = 1024, 1440, 1449
    op = blockops.BlockOperator.from_parallel_beam(n, ang, bins, 8, 8, dtype=np.float32)
    assert 1.8e9 < op.nnz < 2.0e9
    sums = op.matvec(np.ones(n * n), charge=False).reshape(ang, bins)
    offs = np.arange(bins) - (bins - 1) / 2.0
    for a in (0, 1, 360, 719, 1000):
        th = math.pi * a / ang
        c, s = math.cos(th), math.sin(th)
        for b in (0, 100, 724, 1200, bins - 1):
            o = offs[b]
            lo, hi = -1e30, 1e30
            for p0, d in ((o * c, -s if abs(s) >= 1e-12 else 0.0), (o * s, c if abs(c) >= 1e-12 else 0.0)):
                if d == 0.0:
                    if not -n / 2 <= p0 <= n / 2:
                        lo, hi = 0.0, 0.0
                    continue
                t1, t2 = (-n / 2 - p0) / d, (n / 2 - p0) / d
                lo, hi = max(lo, min(t1, t2)), min(hi, max(t1, t2))
            chord = max(0.0, hi - lo)
            assert abs(sums[a, b] - chord) < 1e-3 * max(1.0, chord)   # float32 entries
