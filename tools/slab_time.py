"""Per-rank cost of the slab-decomposed 3-D prox at configs[4] size (256^3).

    python tools/slab_time.py [--iters 10]

One GPU: rank p's slab of P = 1, 2, 4, 8 (an interior slab, so both halos are
live) runs the FGP passes with the host loop's syncs but without peers (the
exchanges are left out: they are measured by NCCL, not here).  Compared with
the single-GPU fused prox kernel on the whole volume.
"""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1812_01307_b200 import parallel, tv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--n", type=int, default=256)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = args.n
    dims = (n, n, n)
    nvox = n ** 3
    rng = np.random.default_rng(0)
    vol = torch.from_numpy(rng.random(nvox)).to(dev)
    g = torch.zeros(nvox, dtype=torch.float64, device=dev)
    w = 0.05
    # single GPU reference: the fused cooperative prox, fixed iterations (tol ~ 0)
    img = vol.view(dims)
    st = tv.ProxSettings(args.iters, 1e-300)
    tv.tv_prox(img, w, st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        tv.tv_prox(img, w, st)
    torch.cuda.synchronize()
    single = (time.perf_counter() - t0) / 3 * 1e3
    print(f"single-GPU fused prox, {args.iters} iterations: {single:.2f} ms")
    for world in (1, 2, 4, 8):
        slabs = parallel.prox_slabs(nvox, world, n * n)
        r = world // 2
        lo, cnt = slabs[r]
        be = parallel.CudaSlab(dims, lo, cnt, dev)
        be.set_weight(w)

        def run():
            be.step(vol, g, 1.0)
            be.init().cpu()
            for _ in range(args.iters):
                be.candidate(False)
                be.dual(0.5).cpu()          # the host loop reads the sums every iteration
                be.parity ^= 1
            be.finalize()
            be.energy().cpu()
        run()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 3 * 1e3
        # per-kernel split of one iteration
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        be.candidate(False)
        ev[1].record()
        be.dual(0.5)
        ev[2].record()
        torch.cuda.synchronize()
        cand, dual = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        print(f"P={world}: slab of {cnt} voxels, {ms:.2f} ms per prox call "
              f"(candidate {cand:.3f} ms + dual {dual:.3f} ms per iteration); "
              f"vs single {single / ms:.2f}x")


if __name__ == "__main__":
    main()
