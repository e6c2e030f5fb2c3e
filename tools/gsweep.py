"""Time configs[1]'s two products for the lanes-per-row choice given by
BSGD_G_FWD / BSGD_G_TR (experiments; the plan's heuristic picks otherwise).

    BSGD_G_TR=16 python tools/gsweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_01307_b200 import _native as nat  # noqa: E402
from paper_1812_01307_b200 import blockops, problems  # noqa: E402

d = problems.config(1)
op = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, 8, 8))
rows, cols = op.shape
x = torch.randn(cols, dtype=torch.float64, device="cuda")
y = torch.randn(rows, dtype=torch.float64, device="cuda")
r = torch.randn(rows, dtype=torch.float64, device="cuda")
ro, g = torch.empty_like(r), torch.empty_like(x)
sp = nat.stream_ptr(op.device)


def t(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


k1 = t(lambda: nat.call("bsgd_residual", op.plan, nat.ptr(x), nat.ptr(y), nat.ptr(ro), None, None, sp))
k2 = t(lambda: nat.call("bsgd_grad", op.plan, nat.ptr(r), nat.ptr(g), sp))
print(f"G_FWD={os.environ.get('BSGD_G_FWD', '-')} G_TR={os.environ.get('BSGD_G_TR', '-')} K1 {k1:.4f} ms K2 {k2:.4f} ms")
