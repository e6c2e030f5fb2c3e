"""Where the host-state (e2e) epoch's time goes on configs[idx]: per-call wall times
of the x / r_vec setters, the epoch and the getters, as bench.py's e2e leg drives them.

    python tools/e2e_prof.py 3
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
    d = problems.config_device(idx)
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=10 ** 9, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    lay = d.layout()
    st = solvers.init_bsgd_state(d.op, d.y, cfg)
    st._ensure_history(256)
    hx = np.zeros(d.op.shape[1])
    hr = np.asarray(d.y.cpu().numpy() if hasattr(d.y, "cpu") else d.y, dtype=np.float64).copy()
    tm = []

    def step():
        nonlocal hx, hr
        t0 = time.perf_counter()
        st.x = hx
        t1 = time.perf_counter()
        st.r_vec = hr
        t2 = time.perf_counter()
        solvers.bsgd_tv_iteration(st, d.op, d.y, cfg, layout=lay)
        t3 = time.perf_counter()
        hx = st.x
        t4 = time.perf_counter()
        hr = st.r_vec
        t5 = time.perf_counter()
        tm.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4))

    for _ in range(5):
        step()
    tm.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        step()
    torch.cuda.synchronize()
    total = (time.perf_counter() - t0) / 20
    a = np.array(tm) * 1e3
    print("set_x set_r epoch get_x get_r (ms):", np.round(a.mean(0), 3), "sum", round(a.sum(1).mean(), 3),
          "wall per epoch", round(total * 1e3, 3))


if __name__ == "__main__":
    main()
