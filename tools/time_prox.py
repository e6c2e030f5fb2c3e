"""Time the TV prox kernel at fixed iteration count (non-converging tol) and report GB/s.

    python tools/time_prox.py [--n 512] [--iters 20] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import tv  # noqa: E402


def prox_bytes(n_pix, iters, restarts=0, dim=2):
    # per FGP iteration of the fused schedule: candidate reads q (dim fields)
    # + b and writes c (dim); dual value + commit reads c, p (2 dim) + b and writes q (dim):
    # 5 dim + 2 field passes; a restart repeats both (5 dim + 2); setup and finalize ~10
    b = 8 * n_pix * ((5 * dim + 2) * (iters + restarts) + 10)
    if n_pix >= (1 << 21) and iters > 0:
        b -= 8 * n_pix * 2 * dim   # split prox: p = q = 0 of the first iteration are not read
    return b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--weight", type=float, default=0.05)
    ap.add_argument("--depth", type=int, default=1, help="> 1: n x n x depth volume (3-D TV)")
    ap.add_argument("--trials", type=int, default=1, help="repeat with a fresh workspace allocation")
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    shape = (a.depth, a.n, a.n) if a.depth > 1 else (a.n, a.n)
    img = torch.tensor(rng.random(shape), device="cuda")
    st = tv.ProxSettings(a.iters, 1e-300)
    out, info = tv.tv_prox(img, a.weight, st, return_info=True)
    torch.cuda.synchronize()
    trials = []
    keep = []
    for _ in range(a.trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            tv.tv_prox(img, a.weight, st)
        e1.record()
        torch.cuda.synchronize()
        trials.append(e0.elapsed_time(e1) / a.reps)
        if a.trials > 1:
            w = next(iter(tv._ws_cache.values()))
            print(f"trial {len(trials)}: ws {w.data_ptr():#x} (mod 1 GiB {w.data_ptr() % (1 << 30):#x}) "
                  f"{trials[-1]:.3f} ms", file=sys.stderr)
        keep.append(tv._ws_cache.copy())   # keep old workspaces alive: the next trial gets new addresses
        tv._ws_cache.clear()
    ms = min(trials)
    b = prox_bytes(img.numel(), info.iterations, info.restarts, len(shape))
    print(json.dumps({"shape": list(shape), "iters": info.iterations, "restarts": info.restarts, "ms": round(ms, 4),
                      "us_per_iter": round(1000 * ms / info.iterations, 2), "bytes": b,
                      "trials_ms": [round(t, 3) for t in trials],
                      "gbs": round(b / (ms * 1e6), 1)}))


if __name__ == "__main__":
    main()
