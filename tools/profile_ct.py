"""Run one CT configuration's epoch products under ncu (plan build excluded).

    ncu --profile-from-start off ... python tools/profile_ct.py [--config 3] [--reps 2]

Builds configs[index] on the device (problems.config_device), then inside a
cudaProfilerStart/Stop window launches the forward product + residual (K1,
`bsgd_residual`) and the transposed product (K2, `bsgd_grad`) `reps` times.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1812_01307_b200 import _native as nat  # noqa: E402
from paper_1812_01307_b200 import problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--time", action="store_true", help="print event-timed ms per product instead")
    ap.add_argument("--fwd-tiles", action="store_true", help="also gather-tile A (4 angles x 4 bins)")
    a = ap.parse_args()
    d = problems.config_device(a.config)
    op = d.op
    if a.fwd_tiles:
        from paper_1812_01307_b200 import blockops
        n, ang, nb, _ = op._slice_source[1]
        op.set_gather_tiles(False, blockops.grid_tiles(ang, nb))
    rows, cols = op.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.rand(cols, dtype=torch.float64, device=dev)
    r = torch.randn(rows, dtype=torch.float64, device=dev)
    y = torch.randn(rows, dtype=torch.float64, device=dev)
    rout = torch.empty_like(r)
    g = torch.empty_like(x)
    sp = nat.stream_ptr(dev)

    def k1():
        nat.call("bsgd_residual", op.plan, nat.ptr(x), nat.ptr(y), nat.ptr(rout), None, None, sp)

    def k2():
        nat.call("bsgd_grad", op.plan, nat.ptr(r), nat.ptr(g), sp)

    for _ in range(2):
        k1(); k2()
    torch.cuda.synchronize()
    if a.time:
        for name, f in (("K1", k1), ("K2", k2)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            print(name, round(e0.elapsed_time(e1) / 10, 4), "ms")
        return
    torch.cuda.profiler.start()
    for _ in range(a.reps):
        k1(); k2()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", rows, cols, op.nnz)


if __name__ == "__main__":
    main()
