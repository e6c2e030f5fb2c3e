"""Sustained throughput of the drop-in `run_solver` on configs[idx]: E epochs by CUDA-graph
replay with the chunked history reads, wall clock included (host sync once per chunk).

    python tools/long_run.py 3 2000
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import problems, solvers, tv  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    d = problems.config_device(idx)
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=epochs, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    prob = solvers.Problem(d.op, d.y, d.x_true, d.layout())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = solvers.run_solver("bsgd", prob, cfg, sample_every=max(1, epochs // 10))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s = tr.samples
    print(f"configs[{idx}]: {epochs} epochs in {dt:.2f} s wall -> {epochs / dt:.1f} epochs/s sustained "
          f"(run_solver, {len(s)} samples)")
    for smp in s[:2] + s[-2:]:
        print(f"   epoch {smp.epoch:7.1f}  rel.err {smp.relative_error:.4e}  objective {smp.objective:.6e}  "
              f"units {smp.matvec_units:.1f}")
    print("   ||x|| =", float(np.linalg.norm(tr.final_x)))


if __name__ == "__main__":
    main()
