"""Run a few BSGD-TV epochs of a configuration for an ncu capture of the
in-epoch kernels (K1 lookahead csr_blocked_kernel, K2 gtile_kernel<..EpiStep>,
the prox), e.g.

    ncu --set full --clock-control none -k regex:csr_blocked -c 1 -o k1 python tools/profile_epoch.py 3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

from paper_1812_01307_b200 import problems, solvers, tv  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    d = problems.config_device(idx)
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=10 ** 9, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    st = solvers.init_bsgd_state(d.op, d.y, cfg)
    lay = d.layout()
    for _ in range(epochs):
        solvers.bsgd_tv_iteration(st, d.op, d.y, cfg, layout=lay)
    torch.cuda.synchronize()
    print("kernels", d.op.kernel_info())


if __name__ == "__main__":
    main()
