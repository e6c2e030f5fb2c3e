"""Eager epochs (with and without the in-epoch phase events) against CUDA-graph replay
of the same epochs on configs[idx]: where the eager path's extra time goes.

    python tools/eager_vs_graph.py 3
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_01307_b200 import problems, solvers, tv  # noqa: E402


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n = 20
    d = problems.config_device(idx)
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=10 ** 9, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    st = solvers.init_bsgd_state(d.op, d.y, cfg)
    st._ensure_history(8 * n + 64)
    lay = d.layout()
    for _ in range(5):
        solvers.bsgd_tv_iteration(st, d.op, d.y, cfg, layout=lay)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def eager(label):
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n):
            solvers.bsgd_tv_iteration(st, d.op, st._y, cfg, layout=lay)
        e1.record()
        torch.cuda.synchronize()
        print(f"{label}: {e0.elapsed_time(e1) / n:.4f} ms/epoch", flush=True)

    eager("eager, no phase events")
    d.op.set_phase_timing(True)
    eager("eager, phase events  ")
    ph, k = d.op.phase_timing()
    d.op.set_phase_timing(False)
    print("   phases", {a: round(b / k, 4) for a, b in ph.items()})
    eager("eager, no phase events")
    runner = solvers._GraphRunner(st, cfg, lay, st._y, 2)
    assert runner.capture(False)
    runner.replay()
    for rep in range(2):
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n // 2):
            runner.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"graph replay          : {e0.elapsed_time(e1) / n:.4f} ms/epoch", flush=True)
    st._rows_used += 2 + 2 * n


if __name__ == "__main__":
    main()
