"""K1 gather-order experiment (BSGD_BLK_ORDER = tile4 | morton): per-phase epoch
times of configs[idx] and the iterate after a few epochs, saved for comparison
between runs with and without the switch.

    BSGD_BLK_ORDER=morton python tools/k1_order.py 3 out_morton.npy
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import problems, solvers, tv  # noqa: E402


def main():
    idx = int(sys.argv[1])
    out = sys.argv[2] if len(sys.argv) > 2 else None
    d = problems.config_device(idx)
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=10 ** 9, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    st = solvers.init_bsgd_state(d.op, d.y, cfg)
    lay = d.layout()
    for _ in range(3):
        solvers.bsgd_tv_iteration(st, d.op, d.y, cfg, layout=lay)
    torch.cuda.synchronize()
    if out:
        np.save(out, st.x)
    d.op.set_phase_timing(True)
    n = 20
    for _ in range(n):
        solvers.bsgd_tv_iteration(st, d.op, d.y, cfg, layout=lay)
    torch.cuda.synchronize()
    ph, n = d.op.phase_timing()
    d.op.set_phase_timing(False)
    print(os.environ.get("BSGD_BLK_ORDER", "none"), d.op.kernel_info(),
          {k: round(v / n, 4) for k, v in ph.items()}, flush=True)


if __name__ == "__main__":
    main()
