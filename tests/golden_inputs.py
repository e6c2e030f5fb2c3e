"""Seeded inputs shared by tests/golden/make_golden.py (which runs the reference on
them) and the tests (which regenerate them instead of storing them)."""

import numpy as np

from paper_1812_01307_b200 import problems


def prox_rows_inputs():
    """Power-of-two images at least 128 wide: the shapes the row-walk 2-D prox
    kernel (csrc/fgp2.cu) serves.  Inputs are regenerated from these seeds by the
    test; only the reference's outputs are stored."""
    rng = np.random.default_rng(2024)
    ph = problems.ellipse_phantom(128, 10, 7)
    return [
        ("ell128", ph + 0.05 * rng.standard_normal((128, 128)), 0.05, 60, 1e-10),
        ("rand128", rng.random((128, 128)) * 2.0, 0.3, 20, 1e-12),
        ("tall256x128", rng.standard_normal((256, 128)), 0.02, 30, 1e-9),
        ("wide128x256", np.kron(rng.random((16, 32)), np.ones((8, 8))) + 0.01 * rng.standard_normal((128, 256)),
         1.0, 15, 1e-5),
    ]
