"""Epoch phases of configs[idx] when the operator is built the reference's way --
`BlockOperator(A_csr, partition)` from a plain host CSR, no grid hints -- beside the
device-generated operator with the sinogram hint.

    python tools/plain_csr_epoch.py 2
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_01307_b200 import blockops, problems, solvers, tv  # noqa: E402


def phases(op, d, mu, lay, n=20):
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=10 ** 9, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    st = solvers.init_bsgd_state(op, d.y, cfg)
    for _ in range(3):
        solvers.bsgd_tv_iteration(st, op, d.y, cfg, layout=lay)
    op.set_phase_timing(True)
    for _ in range(n):
        solvers.bsgd_tv_iteration(st, op, d.y, cfg, layout=lay)
    torch.cuda.synchronize()
    ph, k = op.phase_timing()
    op.set_phase_timing(False)
    return {a: round(b / k, 4) for a, b in ph.items()}


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    d = problems.config_device(idx)
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    lay = d.layout()
    print("hinted   ", d.op.kernel_info(), phases(d.op, d, mu, lay), flush=True)
    csr = d.op.tocsr()
    part = d.op.partition
    d.op._csr = None
    del d.op
    torch.cuda.empty_cache()
    op = blockops.BlockOperator(csr, part)
    print("plain CSR", op.kernel_info(), phases(op, d, mu, lay), flush=True)


if __name__ == "__main__":
    main()
