"""ctypes binding of the C ABI in include/bsgd_b200.h (libbsgd_b200.so).

The shared library is built in-tree by `paper_1812_01307_b200.build` (or
`__graft_entry__.build()`).  There is no fallback: if the library or a CUDA
device is missing, every compute entry point raises instead of silently
running something else.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libbsgd_b200.so")

OK, EINVAL, ECUDA, ENOMEM = 0, 1, 2, 3
F32, F64 = 4, 8
EP_R_NEXT, EP_LOOKAHEAD, EP_MONITOR, EP_SKIP_GRAD, EP_NO_TAIL = 1, 2, 4, 8, 16
H_FNEXT, H_HOLDS, H_XX, H_XE, H_TV, H_PITER, H_PRESTART, H_PCONV, H_PFELL, H_DG, H_DD, H_FCURR = range(12)
HIST_COLS = 12
SCRATCH_BYTES = 65536

c_i64 = ctypes.c_int64
c_p = ctypes.c_void_p


class ProxInfoC(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("fell_back", ctypes.c_int32)]


class SlabArgs(ctypes.Structure):
    """bsgd_slab (include/bsgd_b200.h)."""
    _fields_ = [
        ("depth", c_i64), ("height", c_i64), ("width", c_i64), ("offset", c_i64), ("count", c_i64),
        ("weight", ctypes.c_double), ("parity", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("workspace", c_p), ("workspace_bytes", ctypes.c_size_t),
    ]


SLAB_SLOTS = 12
SLAB_DEVICE, SLAB_MAIN, SLAB_RESTART, SLAB_INTERLEAVED = 1, 1, 2, 8


class KernelInfo(ctypes.Structure):
    """bsgd_kernel_info (include/bsgd_b200.h)."""
    _fields_ = [("fwd_kernel", ctypes.c_int32), ("fwd_lanes", ctypes.c_int32),
                ("tr_kernel", ctypes.c_int32), ("tr_lanes", ctypes.c_int32), ("depth", c_i64),
                ("fwd_order", ctypes.c_int32), ("tr_order", ctypes.c_int32)]


KERNEL_NAMES = {0: "csr", 1: "blocked", 2: "blocked_compressed", 3: "gather_tiled", 4: "stacked",
                5: "stacked_tile"}
GATHER_ORDERS = {0: "native", 1: "tile4", 2: "morton", 4: "tile8x2", 5: "tile2x8"}
TIMING_PHASES = ("k1_first", "k2_step", "prox", "k1_lookahead", "tail")


class EpochArgs(ctypes.Structure):
    _fields_ = [
        ("x_k", c_p), ("r_k", c_p), ("y", c_p), ("g", c_p), ("x_next", c_p), ("r_next", c_p),
        ("r_ahead", c_p), ("x_true", c_p), ("perm", c_p), ("mu", ctypes.c_double),
        ("lam", ctypes.c_double), ("height", c_i64), ("width", c_i64),
        ("max_inner_iters", ctypes.c_int32), ("tol", ctypes.c_double), ("f_curr", c_p),
        ("history", c_p), ("epoch_counter", c_p), ("history_capacity", c_i64),
        ("dual_objectives", c_p), ("workspace", c_p), ("workspace_bytes", ctypes.c_size_t),
        ("flags", ctypes.c_uint32), ("depth", c_i64),
    ]


# name -> (restype, argtypes); mirrors include/bsgd_b200.h
_SIGS = {
    "bsgd_last_error": (ctypes.c_char_p, []),
    "bsgd_version": (ctypes.c_int, []),
    "bsgd_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "bsgd_plan_create": (ctypes.c_int, [ctypes.POINTER(c_p), ctypes.c_int, c_i64, c_i64, c_i64, c_p, c_p, c_p,
                                        ctypes.c_int, c_i64, c_i64, c_p, c_p, c_p]),
    "bsgd_plan_create_device": (ctypes.c_int, [ctypes.POINTER(c_p), ctypes.c_int, c_i64, c_i64, c_i64, c_p, c_p,
                                               c_p, ctypes.c_int, c_i64, c_i64, c_p, c_p, c_p]),
    "bsgd_plan_create_stacked": (ctypes.c_int, [ctypes.POINTER(c_p), ctypes.c_int, c_i64, c_i64, c_i64, c_i64,
                                                c_p, c_p, c_p, ctypes.c_int, c_i64, c_i64, c_p, c_p, c_p]),
    "bsgd_plan_create_stacked_device": (ctypes.c_int, [ctypes.POINTER(c_p), ctypes.c_int, c_i64, c_i64, c_i64,
                                                       c_i64, c_p, c_p, c_p, ctypes.c_int, c_i64, c_i64, c_p, c_p,
                                                       c_p]),
    "bsgd_plan_stacked_info": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p]),
    "bsgd_plan_stacked_tiles": (ctypes.c_int, [c_p, ctypes.c_int, c_i64, c_p, c_p, c_p]),
    "bsgd_plan_gather_tiles": (ctypes.c_int, [c_p, ctypes.c_int, c_i64, c_p, c_p, c_p]),
    "bsgd_plan_blocked_transposed": (ctypes.c_int, [c_p, c_i64, c_i64, c_p]),
    "bsgd_plan_destroy": (ctypes.c_int, [c_p]),
    "bsgd_plan_csr_copy": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p]),
    "bsgd_siddon_csr": (ctypes.c_int, [ctypes.c_int, c_i64, c_i64, c_i64, c_p, c_p, ctypes.c_int,
                                       ctypes.POINTER(c_p), ctypes.POINTER(c_p), ctypes.POINTER(c_p),
                                       ctypes.POINTER(c_i64), c_p]),
    "bsgd_device_free": (ctypes.c_int, [c_p]),
    "bsgd_plan_info": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_plan_kernel_info": (ctypes.c_int, [c_p, ctypes.POINTER(KernelInfo)]),
    "bsgd_plan_set_timing": (ctypes.c_int, [c_p, ctypes.c_int]),
    "bsgd_plan_timing": (ctypes.c_int, [c_p, c_p, c_p]),
    "bsgd_plan_block_nnz": (ctypes.c_int, [c_p, c_i64, c_i64, ctypes.POINTER(c_i64)]),
    "bsgd_plan_block_copy": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "bsgd_plan_transpose_copy": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p]),
    "bsgd_block_matvec": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p, c_p]),
    "bsgd_block_matvec_transpose": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p, c_p]),
    "bsgd_matvec": (ctypes.c_int, [c_p, c_p, c_p, c_p]),
    "bsgd_rmatvec": (ctypes.c_int, [c_p, c_p, c_p, c_p]),
    "bsgd_residual": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_assemble_residual": (ctypes.c_int, [c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "bsgd_pair_products": (ctypes.c_int, [c_p, c_i64, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_tv_prox_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i64]),
    "bsgd_tv_prox": (ctypes.c_int, [c_i64, c_i64, c_p, c_p, ctypes.c_double, ctypes.c_int32, ctypes.c_double,
                                    c_p, ctypes.c_size_t, c_p, c_p, c_p]),
    "bsgd_tv_value": (ctypes.c_int, [c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "bsgd_discrete_gradient": (ctypes.c_int, [c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "bsgd_discrete_divergence": (ctypes.c_int, [c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "bsgd_tv_prox3_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i64, c_i64]),
    "bsgd_tv_prox3": (ctypes.c_int, [c_i64, c_i64, c_i64, c_p, c_p, ctypes.c_double, ctypes.c_int32,
                                     ctypes.c_double, c_p, ctypes.c_size_t, c_p, c_p, c_p]),
    "bsgd_tv_value3": (ctypes.c_int, [c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "bsgd_slab_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i64, c_i64, c_i64]),
    "bsgd_slab_layout": (ctypes.c_int, [c_i64, c_i64, c_i64, c_i64, c_p, c_p]),
    "bsgd_slab_step": (ctypes.c_int, [ctypes.POINTER(SlabArgs), c_p, c_p, ctypes.c_double, c_p]),
    "bsgd_slab_init": (ctypes.c_int, [ctypes.POINTER(SlabArgs), c_p, c_p]),
    "bsgd_slab_candidate": (ctypes.c_int, [ctypes.POINTER(SlabArgs), ctypes.c_int32, c_p]),
    "bsgd_slab_dual": (ctypes.c_int, [ctypes.POINTER(SlabArgs), ctypes.c_double, c_p, c_p]),
    "bsgd_slab_finalize": (ctypes.c_int, [ctypes.POINTER(SlabArgs), c_p]),
    "bsgd_slab_energy": (ctypes.c_int, [ctypes.POINTER(SlabArgs), c_p, c_p]),
    "bsgd_slab_output": (ctypes.c_int, [ctypes.POINTER(SlabArgs), ctypes.c_int32, c_p, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_slab_decide": (ctypes.c_int, [ctypes.POINTER(SlabArgs), ctypes.c_int32, ctypes.c_int32, c_p,
                                        ctypes.c_int32, c_p, ctypes.c_int32, ctypes.c_double, c_p]),
    "bsgd_slab_set_step": (ctypes.c_int, [ctypes.POINTER(SlabArgs), c_i64, ctypes.POINTER(EpochArgs), c_p, c_p]),
    "bsgd_slab_info": (ctypes.c_int, [ctypes.POINTER(SlabArgs), c_p, c_p, c_p]),
    "bsgd_epoch_set_step": (ctypes.c_int, [c_i64, ctypes.POINTER(EpochArgs), c_p, ctypes.c_double, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_p]),
    "bsgd_discrete_gradient3": (ctypes.c_int, [c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_discrete_divergence3": (ctypes.c_int, [c_i64, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_dot": (ctypes.c_int, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_sqdist": (ctypes.c_int, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "bsgd_epoch_workspace_bytes": (ctypes.c_size_t, [c_p, c_i64, c_i64]),
    "bsgd_epoch": (ctypes.c_int, [c_p, ctypes.POINTER(EpochArgs), c_p]),
    "bsgd_grad": (ctypes.c_int, [c_p, c_p, c_p, c_p]),
    "bsgd_step": (ctypes.c_int, [c_i64, ctypes.POINTER(EpochArgs), c_p]),
    "bsgd_epoch_forward": (ctypes.c_int, [c_p, c_p, c_p, c_p, ctypes.POINTER(EpochArgs), c_p]),
    "bsgd_epoch_reduce_forward": (ctypes.c_int, [c_p, ctypes.POINTER(EpochArgs), c_p, c_p]),
    "bsgd_epoch_tail": (ctypes.c_int, [c_p, ctypes.POINTER(EpochArgs), c_p, c_p]),
}

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def load():
    """Load libbsgd_b200.so (raises NativeLibraryMissing if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def declared_symbols():
    return list(_SIGS)


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = load().bsgd_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"bsgd_b200 error {rc}: {msg}")


def call(name: str, *args):
    check(getattr(load(), name)(*args))


# --- torch plumbing -----------------------------------------------------------

def torch():
    import torch as _t
    return _t


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1812_01307_b200 needs a CUDA device (B200); none is visible")
    load()
    if isinstance(device, t.device):
        return t.device("cuda", device.index if device.index is not None else t.cuda.current_device())
    return t.device("cuda", t.cuda.current_device() if device is None else device)


def stream_ptr(device=None) -> int:
    t = torch()
    return t.cuda.current_stream(device).cuda_stream


def ptr(tensor) -> int:
    if tensor is None:
        return None
    return tensor.data_ptr()


def as_f64(t_or_np, device, length=None):
    """Device float64 contiguous tensor from a numpy array / torch tensor (no copy if already so)."""
    t = torch()
    if isinstance(t_or_np, t.Tensor):
        out = t_or_np.to(device=device, dtype=t.float64).contiguous()
    else:
        arr = np.ascontiguousarray(np.asarray(t_or_np, dtype=np.float64))
        out = t.from_numpy(arr).to(device=device, non_blocking=False)
    if length is not None and out.shape != (length,):
        raise ValueError(f"expected vector of length {length}, got {tuple(out.shape)}")
    return out
