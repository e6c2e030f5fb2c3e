"""Isotropic TV on a B200 (drop-in for `bsgdtv.tv`, `pkg/src/bsgdtv/tv.py`).

`ImageGrid`, `PixelLayout` and `ProxSettings` are the reference's host-side
value types (same fields, validation and row-major convention).  `tv_prox`,
`tv_value`, `discrete_gradient` and `discrete_divergence` run as sm_100a
kernels; `tv_prox` is one persistent cooperative kernel
(`csrc/fgp.cuh`) that keeps the FGP restart / stop / fallback decisions on
the device.  `ProxInfo` carries the same diagnostics as the reference.

Volumes (configs[4], 256^3): the reference has 2D TV only.  `VolumeGrid` /
`VolumeLayout` and the 3-D branches of `tv_prox` / `tv_value` extend tv.py's
conventions one axis up (z-major storage, backward differences along z, rows,
columns; dual step 1/(12 w)); the CPU checker is `oracle.tv_prox3`.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat


@dataclass
class ImageGrid:
    """S x T image as a flat row-major float64 vector (`tv.py:28-56`)."""

    height: int
    width: int
    data: np.ndarray

    def __post_init__(self) -> None:
        if self.height < 1 or self.width < 1:
            raise ValueError("image dimensions must be positive")
        self.data = np.asarray(self.data, dtype=np.float64).ravel()
        if self.data.size != self.height * self.width:
            raise ValueError(f"data has {self.data.size} values, expected {self.height * self.width}")

    @classmethod
    def from_matrix(cls, mat) -> "ImageGrid":
        mat = np.asarray(mat, dtype=np.float64)
        if mat.ndim != 2:
            raise ValueError("expected a 2-D array")
        return cls(mat.shape[0], mat.shape[1], mat.ravel().copy())

    def as_matrix(self) -> np.ndarray:
        return self.data.reshape(self.height, self.width)

    def copy(self) -> "ImageGrid":
        return ImageGrid(self.height, self.width, self.data.copy())


@dataclass(frozen=True)
class PixelLayout:
    """Solver-vector position k <-> row-major pixel perm[k] (`tv.py:59-98`)."""

    height: int
    width: int
    perm: np.ndarray

    def __post_init__(self) -> None:
        perm = np.asarray(self.perm, dtype=np.intp)
        n = self.height * self.width
        if perm.shape != (n,) or np.any(np.sort(perm) != np.arange(n)):
            raise ValueError("perm must be a permutation of all pixel indices")
        object.__setattr__(self, "perm", perm)

    @classmethod
    def row_major(cls, height: int, width: int) -> "PixelLayout":
        return cls(height, width, np.arange(height * width, dtype=np.intp))

    @property
    def size(self) -> int:
        return self.height * self.width

    @property
    def is_identity(self) -> bool:
        cached = self.__dict__.get("_is_identity")
        if cached is None:
            cached = bool(np.array_equal(self.perm, np.arange(self.size)))
            object.__setattr__(self, "_is_identity", cached)
        return cached

    def to_image(self, x) -> ImageGrid:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.size,):
            raise ValueError(f"expected vector of length {self.size}, got {x.shape}")
        flat = np.empty(self.size, dtype=np.float64)
        flat[self.perm] = x
        return ImageGrid(self.height, self.width, flat)

    def to_vector(self, img: ImageGrid) -> np.ndarray:
        if (img.height, img.width) != (self.height, self.width):
            raise ValueError("image shape does not match layout")
        return img.data[self.perm].copy()

    def device_perm(self, device):
        """int64 perm on ``device`` (None for the identity layout), cached."""
        if self.is_identity:
            return None
        cache = self.__dict__.setdefault("_dev_perm", {})
        key = str(device)
        if key not in cache:
            t = nat.torch()
            cache[key] = t.from_numpy(self.perm.astype(np.int64)).to(device)
        return cache[key]


@dataclass
class VolumeGrid:
    """D x S x T volume as a flat z-major float64 vector (3-D analogue of `ImageGrid`)."""

    depth: int
    height: int
    width: int
    data: np.ndarray

    def __post_init__(self) -> None:
        if self.depth < 1 or self.height < 1 or self.width < 1:
            raise ValueError("volume dimensions must be positive")
        self.data = np.asarray(self.data, dtype=np.float64).ravel()
        if self.data.size != self.depth * self.height * self.width:
            raise ValueError(f"data has {self.data.size} values, expected {self.depth * self.height * self.width}")

    @classmethod
    def from_array(cls, arr) -> "VolumeGrid":
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 3:
            raise ValueError("expected a 3-D array")
        return cls(arr.shape[0], arr.shape[1], arr.shape[2], arr.ravel().copy())

    def as_array(self) -> np.ndarray:
        return self.data.reshape(self.depth, self.height, self.width)

    def copy(self) -> "VolumeGrid":
        return VolumeGrid(self.depth, self.height, self.width, self.data.copy())


@dataclass(frozen=True)
class VolumeLayout:
    """Solver-vector position k <-> z-major voxel perm[k] (3-D analogue of `PixelLayout`)."""

    depth: int
    height: int
    width: int
    perm: np.ndarray

    def __post_init__(self) -> None:
        perm = np.asarray(self.perm, dtype=np.intp)
        n = self.depth * self.height * self.width
        if perm.shape != (n,) or np.any(np.sort(perm) != np.arange(n)):
            raise ValueError("perm must be a permutation of all voxel indices")
        object.__setattr__(self, "perm", perm)

    @classmethod
    def z_major(cls, depth: int, height: int, width: int) -> "VolumeLayout":
        return cls(depth, height, width, np.arange(depth * height * width, dtype=np.intp))

    @property
    def size(self) -> int:
        return self.depth * self.height * self.width

    is_identity = PixelLayout.is_identity
    device_perm = PixelLayout.device_perm

    def to_image(self, x) -> VolumeGrid:
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.size,):
            raise ValueError(f"expected vector of length {self.size}, got {x.shape}")
        flat = np.empty(self.size, dtype=np.float64)
        flat[self.perm] = x
        return VolumeGrid(self.depth, self.height, self.width, flat)

    def to_vector(self, vol: VolumeGrid) -> np.ndarray:
        if (vol.depth, vol.height, vol.width) != (self.depth, self.height, self.width):
            raise ValueError("volume shape does not match layout")
        return vol.data[self.perm].copy()


def layout_shape(layout) -> tuple:
    """(depth, height, width) of a PixelLayout (depth 1) or VolumeLayout."""
    return (getattr(layout, "depth", 1), layout.height, layout.width)


@dataclass(frozen=True)
class ProxSettings:
    """Inner-solve controls (`tv.py:101-112`)."""

    max_inner_iters: int = 100
    tol: float = 1e-5

    def __post_init__(self) -> None:
        if self.max_inner_iters < 1:
            raise ValueError("max_inner_iters must be >= 1")
        if not self.tol > 0:
            raise ValueError("tol must be positive")


@dataclass
class ProxInfo:
    """Diagnostics from one `tv_prox` call (`tv.py:155-163`)."""

    iterations: int = 0
    converged: bool = False
    restarts: int = 0
    fell_back: bool = False
    dual_objectives: list = field(default_factory=list)


def _image_tensor(img, device):
    """(flat device tensor, shape) with shape (h, w) for images, (d, h, w) for volumes."""
    t = nat.torch()
    if isinstance(img, ImageGrid):
        return nat.as_f64(img.data, device), (img.height, img.width)
    if isinstance(img, VolumeGrid):
        return nat.as_f64(img.data, device), (img.depth, img.height, img.width)
    if isinstance(img, t.Tensor):
        if img.ndim not in (2, 3):
            raise ValueError("expected a 2-D image or 3-D volume tensor")
        return img.to(device=device, dtype=t.float64).contiguous().reshape(-1), tuple(img.shape)
    arr = np.asarray(img, dtype=np.float64)
    if arr.ndim not in (2, 3):
        raise ValueError("expected a 2-D or 3-D array")
    return nat.as_f64(arr.ravel(), device), arr.shape


_ws_cache: dict = {}
_ws_lock = threading.Lock()


def prox_workspace(height: int, width: int, device, depth: int = 1):
    """Zeroed device workspace for `bsgd_tv_prox(3)`, reused across calls of one
    shape on one stream.  The key includes the current CUDA stream and the
    calling thread, so concurrent proxes (other streams or threads) never share
    dual fields or reduction counters; calls on one stream are serialised by
    the stream itself."""
    t = nat.torch()
    dev = t.device(device)
    stream = t.cuda.current_stream(dev).cuda_stream
    key = (depth, height, width, str(dev), stream, threading.get_ident())
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None:
            nbytes = int(nat.load().bsgd_tv_prox3_workspace_bytes(depth, height, width))
            ws = t.zeros((nbytes + 7) // 8, dtype=t.float64, device=dev)
            _ws_cache[key] = ws
    return ws


def _wrap(img, out, shape):
    t = nat.torch()
    if isinstance(img, t.Tensor):
        return out.reshape(shape)
    data = out.cpu().numpy()
    if len(shape) == 3:
        return VolumeGrid(*shape, data)
    return ImageGrid(*shape, data)


def tv_prox(img, weight: float, settings: ProxSettings | None = None, return_info: bool = False):
    """argmin_t ||t - img||^2 + 2 weight TV(t) by restarted dual FGP (`tv.py:172-255`).

    ``img`` may be an `ImageGrid` (result: `ImageGrid`), a `VolumeGrid`
    (result: `VolumeGrid`, 3-D TV) or a 2-D / 3-D CUDA tensor (result:
    tensor).  weight = 0 is the identity; weight < 0 raises.
    """
    if weight < 0:
        raise ValueError("prox weight must be nonnegative")
    if settings is None:
        settings = ProxSettings()
    t = nat.torch()
    device = img.device if isinstance(img, t.Tensor) and img.is_cuda else nat.require_cuda()
    b, shape = _image_tensor(img, device)
    out = t.empty_like(b)
    info_dev = t.zeros(4, dtype=t.int32, device=device)
    dual = t.empty(settings.max_inner_iters + 1, dtype=t.float64, device=device) if return_info else None
    common = (nat.ptr(b), nat.ptr(out), float(weight), int(settings.max_inner_iters), float(settings.tol))
    if len(shape) == 3:
        d, h, w = shape
        ws = prox_workspace(h, w, device, depth=d)
        nat.call("bsgd_tv_prox3", d, h, w, *common, nat.ptr(ws), ws.numel() * 8, nat.ptr(info_dev),
                 nat.ptr(dual), nat.stream_ptr(device))
    else:
        h, w = shape
        ws = prox_workspace(h, w, device)
        nat.call("bsgd_tv_prox", h, w, *common, nat.ptr(ws), ws.numel() * 8, nat.ptr(info_dev), nat.ptr(dual),
                 nat.stream_ptr(device))
    result = _wrap(img, out, shape)
    if not return_info:
        return result
    it, conv, rst, fell = (int(v) for v in info_dev.cpu().tolist())
    info = ProxInfo(iterations=it, converged=bool(conv), restarts=rst, fell_back=bool(fell))
    if weight == 0.0:
        info.dual_objectives = []
    else:
        info.dual_objectives = dual[: it + 1].cpu().tolist()
    return result, info


def tv_value(img) -> float:
    """Isotropic TV (`tv.py:149-152`; volumes: the 3-D extension), reduced on the device."""
    t = nat.torch()
    device = img.device if isinstance(img, t.Tensor) and img.is_cuda else nat.require_cuda()
    b, shape = _image_tensor(img, device)
    scratch = t.empty(nat.SCRATCH_BYTES // 8, dtype=t.float64, device=device)
    out = t.empty(1, dtype=t.float64, device=device)
    if len(shape) == 3:
        nat.call("bsgd_tv_value3", *shape, nat.ptr(b), nat.ptr(out), nat.ptr(scratch), nat.stream_ptr(device))
    else:
        nat.call("bsgd_tv_value", *shape, nat.ptr(b), nat.ptr(out), nat.ptr(scratch), nat.stream_ptr(device))
    return float(out.item())


def discrete_gradient(img: ImageGrid):
    """(vertical, horizontal) backward differences, zero on row / column 0 (`tv.py:135-137`)."""
    t = nat.torch()
    device = nat.require_cuda()
    b, (h, w) = _image_tensor(img, device)
    dv = t.empty_like(b)
    dh = t.empty_like(b)
    nat.call("bsgd_discrete_gradient", h, w, nat.ptr(b), nat.ptr(dv), nat.ptr(dh), nat.stream_ptr(device))
    return dv.reshape(h, w).cpu().numpy(), dh.reshape(h, w).cpu().numpy()


def discrete_divergence(pv, ph) -> ImageGrid:
    """Negative adjoint of `discrete_gradient` (`tv.py:140-146`)."""
    pv = np.asarray(pv, dtype=np.float64)
    ph = np.asarray(ph, dtype=np.float64)
    if pv.shape != ph.shape or pv.ndim != 2:
        raise ValueError("difference fields must be two equal-shape 2-D arrays")
    t = nat.torch()
    device = nat.require_cuda()
    a = nat.as_f64(pv.ravel(), device)
    b = nat.as_f64(ph.ravel(), device)
    out = t.empty_like(a)
    nat.call("bsgd_discrete_divergence", pv.shape[0], pv.shape[1], nat.ptr(a), nat.ptr(b), nat.ptr(out),
             nat.stream_ptr(device))
    return ImageGrid(pv.shape[0], pv.shape[1], out.cpu().numpy())


def discrete_gradient3(vol):
    """(z, vertical, horizontal) backward differences of a volume, zero on the first slice / row / column."""
    t = nat.torch()
    device = nat.require_cuda()
    b, shape = _image_tensor(vol, device)
    if len(shape) != 3:
        raise ValueError("expected a volume")
    dz, dv, dh = (t.empty_like(b) for _ in range(3))
    nat.call("bsgd_discrete_gradient3", *shape, nat.ptr(b), nat.ptr(dz), nat.ptr(dv), nat.ptr(dh),
             nat.stream_ptr(device))
    return tuple(f.reshape(shape).cpu().numpy() for f in (dz, dv, dh))


def discrete_divergence3(pz, pv, ph) -> VolumeGrid:
    """Negative adjoint of `discrete_gradient3`."""
    fields = [np.asarray(f, dtype=np.float64) for f in (pz, pv, ph)]
    if fields[0].ndim != 3 or any(f.shape != fields[0].shape for f in fields):
        raise ValueError("difference fields must be three equal-shape 3-D arrays")
    t = nat.torch()
    device = nat.require_cuda()
    devs = [nat.as_f64(f.ravel(), device) for f in fields]
    out = t.empty_like(devs[0])
    nat.call("bsgd_discrete_divergence3", *fields[0].shape, *(nat.ptr(d) for d in devs), nat.ptr(out),
             nat.stream_ptr(device))
    return VolumeGrid(*fields[0].shape, out.cpu().numpy())
