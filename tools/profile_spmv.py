"""Run the configs[1] SpMV kernels (K1 forward+residual, K2 transposed) a few times for ncu.

    python tools/profile_spmv.py [--reps 3] [--config 1] [--scale 1.0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1812_01307_b200 import _native as nat  # noqa: E402
from paper_1812_01307_b200 import blockops, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    d = problems.config(a.config, scale=a.scale)
    m = d.num_row_blocks
    op = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, m, m))
    dev = op.device
    rows, cols = op.shape
    x = torch.randn(cols, dtype=torch.float64, device=dev)
    r = torch.randn(rows, dtype=torch.float64, device=dev)
    y = torch.randn(rows, dtype=torch.float64, device=dev)
    rout = torch.empty_like(r)
    g = torch.empty_like(x)
    sp = nat.stream_ptr(dev)
    for _ in range(a.reps):
        nat.call("bsgd_residual", op.plan, nat.ptr(x), nat.ptr(y), nat.ptr(rout), None, None, sp)
        nat.call("bsgd_grad", op.plan, nat.ptr(r), nat.ptr(g), sp)
    torch.cuda.synchronize()
    print("ok", rows, cols, op.nnz)


if __name__ == "__main__":
    main()
