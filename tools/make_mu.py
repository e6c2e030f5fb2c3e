"""Compute the step mu = 0.9 / (2 u_max) of every BASELINE.json configuration ONCE
and record it in tests/golden/config_mu.json, so that bench.py's two arms (the
B200 path and the CPU reference) and the full-size parity tests all run with
the identical float64 mu.

u_max comes from `spectral.largest_eigenvalue(op, max_iters=50)` on the GPU
(the reference's power iteration, `spectral.py:43-75`, same seeded start
vector and stop rule; within 1e-10 of the reference's value, tests/
test_gpu_kernels.py).  The CPU reference would take ~100 s per config for
the same 50 iterations at configs[3].

    gpurun -- python tools/make_mu.py [index ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
OUT = os.path.join(REPO, "tests", "golden", "config_mu.json")


def main(indices):
    import torch

    from paper_1812_01307_b200 import blockops, problems, spectral

    table = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            table = json.load(fh)
    for idx in indices:
        t0 = time.time()
        if idx == 1:
            d = problems.config(1)
            op = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.matrix.shape, 8, 8))
        else:
            op = problems.config_device(idx).op
        pw = spectral.largest_eigenvalue(op, max_iters=50)
        table[f"configs[{idx}]"] = {"u_max": pw.value, "mu": 0.9 / (2.0 * pw.value), "converged": pw.converged,
                                    "iterations": pw.iterations, "shape": list(op.shape), "nnz": int(op.nnz),
                                    "how": "spectral.largest_eigenvalue(op, max_iters=50) on a B200, seed 0"}
        print(f"configs[{idx}]: u_max={pw.value!r} mu={0.9 / (2.0 * pw.value)!r} ({time.time() - t0:.1f}s)",
              flush=True)
        del op
        torch.cuda.empty_cache()
    with open(OUT, "w") as fh:
        json.dump(table, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4])
