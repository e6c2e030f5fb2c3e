"""One rank's share of a configs[3] epoch at N = 1, 2, 4, 8 ranks, measured on ONE GPU.

Rank 0's row slab (its 1/N of the angles, generated on the device) runs the real
`DistributedBSGD` epoch with no process group: its products on its own rays plus the
replicated step, prox and tail -- everything a rank computes between two all-reduces.
The collective itself is NOT included (only one GPU is reachable), and the iterate
follows the rank's partial gradient, so this bounds the scaling from above:

    epochs/s at N ranks <= 1 / (t_rank(N) + t_allreduce(8 MB))

    python tools/rank_share.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import parallel, problems, solvers, tv  # noqa: E402
from paper_1812_01307_b200.blockops import make_partition  # noqa: E402


def main():
    idx = 3
    name, n, ang, nb, ell, noise_frac, blocks, lam, inner, epochs, dt = problems.CT_TABLE[idx]
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                           "config_mu.json")) as fh:
        mu = json.load(fh)[f"configs[{idx}]"]["mu"]
    d = problems.config_device(idx)
    y_full = np.asarray(d.y.cpu().numpy() if hasattr(d.y, "cpu") else d.y, dtype=np.float64)
    del d
    torch.cuda.empty_cache()
    part = make_partition(ang * nb, n * n, blocks, blocks)
    layout = tv.PixelLayout.row_major(n, n)
    cfg = solvers.SolverConfig(mu=mu, lam=lam, epochs=10 ** 9, prox=tv.ProxSettings(inner, 1e-5),
                               monitor_decrease=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    base = None
    for world in (1, 2, 4, 8):
        shard = parallel.CudaShard.parallel_beam(n, ang, nb, parallel.ShardSpec(part, 0, world), dtype=dt, lam=lam,
                                                 layout=layout)
        drv = parallel.DistributedBSGD(shard, y_full, cfg, history_capacity=256, prox="replicated")
        for _ in range(4):
            drv.epoch_step()
        steps = 20
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            drv.epoch_step()
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / steps
        graph = float("nan")
        if drv.capture(2):
            drv.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(steps // 2):
                drv.replay()
            e1.record()
            torch.cuda.synchronize()
            graph = e0.elapsed_time(e1) / steps
        t = min(eager, graph) if graph == graph else eager
        base = base or t
        print(f"N={world}: rank 0 owns {shard.rows} rays ({shard.op.nnz / 1e6:.0f}M nnz): eager {eager:.4f} ms, "
              f"graph {graph:.4f} ms per epoch -> compute-only bound {1000.0 / t:.0f} epochs/s "
              f"({base / t:.2f}x of N=1, {base / t / world:.2f} efficiency before the all-reduce)", flush=True)
        del drv, shard
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
