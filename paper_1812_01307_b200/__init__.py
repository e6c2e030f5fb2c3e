"""B200-native drop-in for the BSGD-TV epoch path of the `bsgdtv` reference (arXiv 1812.01307).

Modules mirror the reference package (`pkg/src/bsgdtv/`): `blockops`, `tv`,
`solvers`, `metrics`, `spectral`; `parallel` adds the multi-GPU row-slab
ownership and `problems` the seeded benchmark inputs.  Compute runs in
`lib/libbsgd_b200.so` (sm_100a CUDA behind the C ABI of include/bsgd_b200.h).
"""

__version__ = "0.1.0"
