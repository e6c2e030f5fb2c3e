"""configs[2]/[3] products with and without gather tiles: python tools/gtile_sweep.py [index]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import _native as nat  # noqa: E402
from paper_1812_01307_b200 import blockops  # noqa: E402

geo = {2: (512, 720, 727), 3: (1024, 1440, 1449)}[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
n, ang, nb = geo
out = {"n": n}
for tiles in (False, True):
    op = blockops.BlockOperator.from_parallel_beam(n, ang, nb, 8, 8, dtype=np.float32, tiles=tiles)
    rows, cols = op.shape
    torch.manual_seed(0)
    x = torch.rand(cols, dtype=torch.float64, device="cuda")
    r = torch.rand(rows, dtype=torch.float64, device="cuda")
    yo = torch.empty(rows, dtype=torch.float64, device="cuda")
    go = torch.empty(cols, dtype=torch.float64, device="cuda")
    st = nat.stream_ptr()
    res = {}
    for name, fn, o in (("k1", lambda: nat.call("bsgd_matvec", op.plan, nat.ptr(x), nat.ptr(yo), st), yo),
                        ("k2", lambda: nat.call("bsgd_rmatvec", op.plan, nat.ptr(r), nat.ptr(go), st), go)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_ms"] = round(e0.elapsed_time(e1) / 10, 4)
        res[name] = o.clone()
    out["tiles" if tiles else "csr"] = {k: v for k, v in res.items() if k.endswith("_ms")}
    if tiles:
        out["k1_rel"] = float(((res["k1"] - prev["k1"]).norm() / prev["k1"].norm()).item())
        out["k2_rel"] = float(((res["k2"] - prev["k2"]).norm() / prev["k2"].norm()).item())
    prev = res
print(json.dumps(out))
