"""Compare the panel-tiled SpMV with the CSR kernels and time both (configs[1]).

    python tools/check_tiled.py [--scale S] [--config I] [--time]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import _native as nat  # noqa: E402
from paper_1812_01307_b200 import blockops, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.05)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--profile", action="store_true", help="3 tiled launches of each kernel only")
    a = ap.parse_args()
    d = problems.config(a.config, scale=a.scale)
    m = d.num_row_blocks
    os.environ["BSGD_TILED"] = "1"
    t0 = time.time()
    op_t = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, m, m))
    torch.cuda.synchronize()
    print(f"tiled plan {time.time() - t0:.2f}s", flush=True)
    if a.profile:
        x = torch.randn(d.shape[1], dtype=torch.float64, device="cuda")
        w = torch.randn(d.shape[0], dtype=torch.float64, device="cuda")
        for _ in range(3):
            op_t.matvec(x)
            op_t.rmatvec(w)
        torch.cuda.synchronize()
        print("profiled")
        return
    os.environ["BSGD_TILED"] = "0"
    op_c = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, m, m))
    rng = np.random.default_rng(0)
    x = torch.tensor(rng.standard_normal(d.shape[1]), device="cuda")
    w = torch.tensor(rng.standard_normal(d.shape[0]), device="cuda")
    for name, ft, fc in [("matvec", lambda: op_t.matvec(x), lambda: op_c.matvec(x)),
                         ("rmatvec", lambda: op_t.rmatvec(w), lambda: op_c.rmatvec(w))]:
        yt, yc = ft(), fc()
        torch.cuda.synchronize()
        err = (torch.linalg.norm(yt - yc) / torch.linalg.norm(yc)).item()
        print(f"{name}: rel diff tiled vs csr = {err:.3e}", flush=True)
        assert err < 1e-12, err
        if a.time:
            for label, f in (("tiled", ft), ("csr", fc)):
                for _ in range(3):
                    f()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    f()
                e1.record()
                torch.cuda.synchronize()
                print(f"  {label:6s} {e0.elapsed_time(e1) / 20:.4f} ms", flush=True)
    print("ok")


if __name__ == "__main__":
    main()
