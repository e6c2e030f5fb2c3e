"""Time the slice-stacked products (K1 forward, K2 transposed) of configs[4] at full size.

    BSGD_STK_L2_BYTES=... python tools/stk_sweep.py [--scale 1.0]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import _native as nat  # noqa: E402
from paper_1812_01307_b200 import blockops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--depth", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    op = blockops.BlockOperator.from_parallel_beam(a.n, 360 * a.n // 256, (363 * a.n // 256) | 1, 16, 16, tiles=not os.environ.get("STK_NO_TILES"),
                                                   dtype=np.float32, depth=a.depth)
    rows, cols = op.shape
    x = torch.rand(cols, dtype=torch.float64, device="cuda")
    r = torch.rand(rows, dtype=torch.float64, device="cuda")
    yo = torch.empty(rows, dtype=torch.float64, device="cuda")
    go = torch.empty(cols, dtype=torch.float64, device="cuda")
    st = nat.stream_ptr()
    out = {"env": os.environ.get("BSGD_STK_L2_BYTES"), "nnz": op.nnz}
    for name, fn in (("k1", lambda: nat.call("bsgd_matvec", op.plan, nat.ptr(x), nat.ptr(yo), st)),
                     ("k2", lambda: nat.call("bsgd_rmatvec", op.plan, nat.ptr(r), nat.ptr(go), st))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        out[name + "_ms"] = round(ms, 3)
        out[name + "_l2_gbs"] = round(op.nnz * 8 / (ms * 1e6), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
