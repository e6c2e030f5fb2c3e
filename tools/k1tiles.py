import sys, os, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1812_01307_b200 import blockops, _native as nat
for idx, (n, ang, nb) in ((2, (512, 720, 727)), (3, (1024, 1440, 1449))):
    op = blockops.BlockOperator.from_parallel_beam(n, ang, nb, 8, 8, dtype=np.float32, tiles=False)
    rows, cols = op.shape
    x = torch.rand(cols, dtype=torch.float64, device="cuda"); yo = torch.empty(rows, dtype=torch.float64, device="cuda")
    st = nat.stream_ptr()
    def t():
        f = lambda: nat.call("bsgd_matvec", op.plan, nat.ptr(x), nat.ptr(yo), st)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / 10, 4)
    res = {"csr": t()}
    for th, tw in ((4, 4), (2, 8), (8, 2), (16, 1), (1, 16)):
        op.set_gather_tiles(False, blockops.grid_tiles(ang, nb, th, tw))
        res[f"{th}x{tw}"] = t()
    print(idx, json.dumps(res))
