"""Reconstruction metrics on the device (drop-in for `bsgdtv.metrics`, `metrics.py:11-38`)."""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .blockops import BlockOperator
from .tv import PixelLayout, layout_shape, tv_value


def _dev_of(*vals):
    t = nat.torch()
    for v in vals:
        if isinstance(v, t.Tensor) and v.is_cuda:
            return v.device
    return nat.require_cuda()


def relative_error(x, x_true) -> float:
    """||x - x_true|| / ||x_true|| (`metrics.py:11-20`); ValueError for a zero reference."""
    t = nat.torch()
    dev = _dev_of(x, x_true)
    xv = nat.as_f64(x, dev)
    tv_ = nat.as_f64(x_true, dev)
    if xv.shape != tv_.shape:
        raise ValueError(f"shape mismatch: {tuple(xv.shape)} vs {tuple(tv_.shape)}")
    scratch = t.empty(nat.SCRATCH_BYTES // 8, dtype=t.float64, device=dev)
    out = t.empty(2, dtype=t.float64, device=dev)
    n = xv.numel()
    nat.call("bsgd_dot", n, nat.ptr(tv_), nat.ptr(tv_), nat.ptr(out[0:1]), nat.ptr(scratch), nat.stream_ptr(dev))
    nat.call("bsgd_sqdist", n, nat.ptr(xv), nat.ptr(tv_), nat.ptr(out[1:2]), nat.ptr(scratch),
             nat.stream_ptr(dev))
    den2, num2 = (float(v) for v in out.cpu().tolist())
    if den2 == 0.0:
        raise ValueError("reference vector is zero; relative error undefined")
    return float(np.sqrt(num2) / np.sqrt(den2))


def objective_value(x, op: BlockOperator, y, lam: float, layout: PixelLayout | None = None,
                    charge: bool = True) -> float:
    """||y - A x||^2 + 2 lam TV(image of x) (`metrics.py:23-38`); charges one unit."""
    if lam < 0:
        raise ValueError("lam must be nonnegative")
    _, s = op.residual_sumsq(x, y, charge=charge)
    value = float(s.item())
    if lam > 0:
        if layout is None:
            raise ValueError("layout required to evaluate the TV term")
        t = nat.torch()
        xv = nat.as_f64(x, op.device, layout.size)
        perm = layout.device_perm(op.device)
        img = xv if perm is None else t.empty_like(xv).index_copy_(0, perm, xv)
        value += 2.0 * lam * tv_value(img.reshape(layout_shape(layout) if hasattr(layout, "depth") else (layout.height, layout.width)))
    return value
