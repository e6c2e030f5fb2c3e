"""3-D isotropic TV on the GPU (configs[4]) against the oracle's 3-D restatement.

The reference has 2D TV only, so this extension is PARITY UNPINNED against
the reference itself; `oracle.tv_prox3` is its checker.  The
device kernel is the 2D kernel templated over the dimension, with the same
op-for-op rounding and numpy-order pairwise sums, so agreement is bit-exact:
outputs, ProxInfo and dual objectives.
"""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tv(cuda_ok):
    from paper_1812_01307_b200 import tv as _tv
    return _tv


@pytest.mark.parametrize("shape,w,iters", [((4, 3, 5), 0.3, 20), ((8, 12, 16), 0.05, 20), ((16, 16, 16), 0.02, 20),
                                           ((2, 64, 64), 0.1, 10), ((32, 32, 32), 0.01, 10),
                                           ((5, 40, 7), 1e-3, 30), ((64, 128, 128), 0.02, 8),
                                           ((100, 100, 100), 0.05, 6)])
def test_tv_prox3_bit_exact(tv, shape, w, iters):
    vol = np.random.default_rng(sum(shape)).random(shape) * 2.0
    out, info = tv.tv_prox(tv.VolumeGrid.from_array(vol), w, tv.ProxSettings(iters, 1e-12), return_info=True)
    ref, rep = orc.tv_prox3(vol, w, iters, 1e-12)
    assert np.array_equal(out.as_array(), ref)
    assert (info.iterations, info.converged, info.restarts, info.fell_back) == \
        (rep.iterations, rep.converged, rep.restarts, rep.fell_back)
    assert np.array_equal(np.array(info.dual_objectives), np.array(rep.dual_objectives))


def test_tv_prox3_stops_and_falls_back(tv):
    rng = np.random.default_rng(11)
    vol = rng.random((6, 9, 10))
    # loose tolerance: early stop on the relative-change test
    out, info = tv.tv_prox(tv.VolumeGrid.from_array(vol), 0.02, tv.ProxSettings(200, 1e-2), return_info=True)
    ref, rep = orc.tv_prox3(vol, 0.02, 200, 1e-2)
    assert rep.converged and info.converged and info.iterations == rep.iterations < 200
    assert np.array_equal(out.as_array(), ref)
    # huge weight, one iteration: the identity fallback decides the same way
    out, info = tv.tv_prox(tv.VolumeGrid.from_array(vol), 50.0, tv.ProxSettings(1, 1e-12), return_info=True)
    ref, rep = orc.tv_prox3(vol, 50.0, 1, 1e-12)
    assert info.fell_back == rep.fell_back
    assert np.array_equal(out.as_array(), ref)


def test_tv_prox3_edge_cases(tv):
    vol = tv.VolumeGrid.from_array(np.random.default_rng(0).random((3, 5, 6)))
    same, info = tv.tv_prox(vol, 0.0, return_info=True)
    assert np.array_equal(same.data, vol.data) and info.converged and info.iterations == 0
    const = tv.VolumeGrid.from_array(np.full((4, 7, 7), 5.0))
    assert np.array_equal(tv.tv_prox(const, 0.7).data, const.data)
    with pytest.raises(ValueError):
        tv.tv_prox(vol, -1.0)


def test_tv_prox3_tensor_in_tensor_out(tv):
    import torch
    vol = np.random.default_rng(3).random((4, 16, 16))
    got = tv.tv_prox(torch.from_numpy(vol).cuda(), 0.1, tv.ProxSettings(15, 1e-12))
    assert got.shape == (4, 16, 16) and got.is_cuda
    ref, _ = orc.tv_prox3(vol, 0.1, 15, 1e-12)
    assert np.array_equal(got.cpu().numpy(), ref)


def test_tv_value3_and_difference_operators(tv):
    rng = np.random.default_rng(5)
    vol = rng.random((5, 7, 9))
    assert tv.tv_value(tv.VolumeGrid.from_array(vol)) == orc.tv_value3(vol)
    big = rng.random((64, 64, 64))
    assert tv.tv_value(tv.VolumeGrid.from_array(big)) == orc.tv_value3(big)
    dz, dv, dh = tv.discrete_gradient3(tv.VolumeGrid.from_array(vol))
    rz, rv, rh = orc.forward_diff3(vol)
    assert np.array_equal(dz, rz) and np.array_equal(dv, rv) and np.array_equal(dh, rh)
    p = [rng.standard_normal(vol.shape) for _ in range(3)]
    div = tv.discrete_divergence3(*p).as_array()
    assert np.array_equal(div, orc.divergence3(*p))
    # adjointness <grad u, p> = -<u, div p>
    lhs = sum(float(np.sum(a * b)) for a, b in zip((dz, dv, dh), p))
    assert lhs == pytest.approx(-float(np.sum(vol * div)), rel=1e-12)


@pytest.mark.parametrize("shape,w,iters", [((2048, 2048), 0.05, 4), ((128, 128, 128), 0.05, 3),
                                           ((4, 1024, 512), 0.1, 3)])
def test_prox_direct_leaf_sums_bit_exact(tv, shape, w, iters):
    """Sizes whose numpy-order sums take the barrier-free direct leaf path
    (pairwise.cuh pw_cta_direct): the cooperative kernel at 2048^2 (128 leaves per
    CTA) and the split prox at >= 2^21 voxels (512 CTAs)."""
    arr = np.random.default_rng(len(shape) * 7 + iters).random(shape) * 2.0
    if len(shape) == 2:
        import torch
        out, info = tv.tv_prox(torch.tensor(arr, device="cuda"), w, tv.ProxSettings(iters, 1e-12), return_info=True)
        ref, rep = orc.tv_prox(arr, w, iters, 1e-12)
        got = out.cpu().numpy()
    else:
        out, info = tv.tv_prox(tv.VolumeGrid.from_array(arr), w, tv.ProxSettings(iters, 1e-12), return_info=True)
        ref, rep = orc.tv_prox3(arr, w, iters, 1e-12)
        got = out.as_array()
    assert np.array_equal(got, ref)
    assert (info.iterations, info.restarts, info.fell_back) == (rep.iterations, rep.restarts, rep.fell_back)
    assert np.array_equal(np.array(info.dual_objectives), np.array(rep.dual_objectives))
