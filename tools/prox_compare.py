"""Time the 2-D TV prox kernels at a fixed FGP iteration count (non-converging
tol): the row-walk kernel (default for power-of-two images <= 1024 wide) against
the cooperative fgp_kernel<2> (BSGD_PROX_KERNEL=coop).

    python tools/prox_compare.py [--sizes 512 1024] [--iters 20] [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_01307_b200 import tv  # noqa: E402


def time_prox(img, w, st, reps):
    tv.tv_prox(img, w, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tv.tv_prox(img, w, st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[512, 1024])
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--weight", type=float, default=0.05)
    a = ap.parse_args()
    st = tv.ProxSettings(a.iters, 1e-300)
    for n in a.sizes:
        g = torch.Generator(device="cuda").manual_seed(n)
        img = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g)
        res = {"n": n, "iters": a.iters}
        for kernel in ("rows", "coop"):
            if kernel == "coop":
                os.environ["BSGD_PROX_KERNEL"] = "coop"
            else:
                os.environ.pop("BSGD_PROX_KERNEL", None)
            res[kernel + "_ms"] = round(time_prox(img, a.weight, st, a.reps), 4)
        os.environ.pop("BSGD_PROX_KERNEL", None)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
