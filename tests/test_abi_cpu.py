"""The C-ABI library loads and exports every symbol the header declares (no GPU needed)."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "bsgd_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bsgd_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1812_01307_b200 import _native, build
    build.build()
    return _native.load()


def test_every_declared_symbol_is_exported(lib):
    names = header_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    from paper_1812_01307_b200 import _native
    assert sorted(_native.declared_symbols()) == header_functions()


def test_host_only_entry_points(lib):
    from paper_1812_01307_b200 import _native as nat
    assert lib.bsgd_version() >= 100
    n = ctypes.c_int(-1)
    assert lib.bsgd_device_count(ctypes.byref(n)) == 0
    assert n.value >= 0
    assert lib.bsgd_tv_prox_workspace_bytes(16, 16) > 6 * 256 * 8
    assert lib.bsgd_tv_prox_workspace_bytes(0, 16) == 0
    assert lib.bsgd_epoch_workspace_bytes(None, 4, 4) == 0
    # argument validation happens before any device work
    rc = lib.bsgd_tv_prox(4, 4, None, None, 1.0, 5, 1e-5, None, 0, None, None, None)
    assert rc == nat.EINVAL
    with pytest.raises(ValueError, match="NULL image"):
        nat.check(rc)
    rc = lib.bsgd_tv_prox(4, 4, ctypes.c_void_p(8), ctypes.c_void_p(8), -1.0, 5, 1e-5, None, 0, None, None, None)
    assert rc == nat.EINVAL and b"nonnegative" in lib.bsgd_last_error()
    rc = lib.bsgd_assemble_residual(0, 1, None, None, None, None)
    assert rc == nat.EINVAL


def test_plan_create_validates_before_touching_a_device(lib):
    import numpy as np
    from paper_1812_01307_b200 import _native as nat
    h = nat.c_p()
    indptr = np.array([0, 1, 2], dtype=np.int64)
    idx = np.array([0, 1], dtype=np.int32)
    val = np.array([1.0, 2.0])
    rb = np.array([0, 2], dtype=np.int64)
    cb = np.array([0, 2], dtype=np.int64)
    args = [ctypes.byref(h), 0, 2, 2, 2, indptr.ctypes.data, idx.ctypes.data, val.ctypes.data, 8, 1, 1,
            rb.ctypes.data, cb.ctypes.data, None]
    bad = list(args)
    bad[4] = 0  # nnz == 0 -> ValueError like blockops.py:127-128
    assert lib.bsgd_plan_create(*bad) == nat.EINVAL
    assert b"no nonzeros" in lib.bsgd_last_error()
    bad = list(args)
    bad[8] = 2  # dtype
    assert lib.bsgd_plan_create(*bad) == nat.EINVAL
    bad = list(args)
    bad[9] = 3  # more row blocks than rows
    assert lib.bsgd_plan_create(*bad) == nat.EINVAL
    rc = lib.bsgd_plan_create(*args)
    assert rc in (nat.OK, nat.ECUDA)  # ECUDA when there is no device (this container)
    if rc == nat.OK:
        lib.bsgd_plan_destroy(h)


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from scipy import sparse
    from paper_1812_01307_b200 import blockops
    with pytest.raises(RuntimeError, match="CUDA device"):
        blockops.BlockOperator(sparse.eye(4, format="csr"))
