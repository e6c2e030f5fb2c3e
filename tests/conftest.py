import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def golden_cfg(z):
    return json.loads(bytes(z["cfg"]).decode())


def golden_csr(z):
    from scipy import sparse
    shape = tuple(int(v) for v in z["shape"])
    return sparse.csr_array((z["data"], z["indices"], z["indptr"]), shape=shape)


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
