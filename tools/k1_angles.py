"""K1 (A x) and K2 (A^T r) per angle range and gather order on the configs[3] geometry:
does a ray's / pixel's best gather order depend on the ray direction?

    BSGD_BLK_ORDER=native python tools/k1_angles.py        (or tile4)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_01307_b200 import blockops  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n, ang, nb = 1024, 1440, 1449
    order = os.environ.get("BSGD_BLK_ORDER", "tile4")
    for a0, a1 in ((0, 90), (135, 225), (315, 405), (495, 585), (675, 765), (1035, 1125)):
        op = blockops.BlockOperator.from_parallel_beam(n, ang, nb, 1, 1, angle_range=(a0, a1))
        rows, cols = op.shape
        x = torch.rand(cols, dtype=torch.float64, device="cuda")
        r = torch.rand(rows, dtype=torch.float64, device="cuda")
        t1 = timeit(lambda: op.matvec(x, charge=False))
        t2 = timeit(lambda: op.rmatvec(r, charge=False))
        ki = op.kernel_info()
        print(f"{order:7s} angles [{a0:4d},{a1:4d}) theta {180.0 * a0 / ang:5.1f}-{180.0 * a1 / ang:5.1f} deg  nnz {op.nnz / 1e6:6.1f}M  "
              f"K1 {t1:.4f} ms ({op.nnz * 8 / t1 / 1e6:6.0f} GB/s model)  K2 {t2:.4f} ms ({op.nnz * 8 / t2 / 1e6:6.0f})  "
              f"{ki['forward']}/{ki['forward_lanes']}/{ki['forward_order']} {ki['transposed']}/{ki['transposed_order']}",
              flush=True)
        del op
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
