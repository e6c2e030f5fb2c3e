"""Repeat the 3-D prox with fresh workspaces and record SM clock / throttle reasons per trial (NVML)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1812_01307_b200 import tv  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
img = torch.tensor(np.random.default_rng(0).random((256, 256, 256)), device="cuda")
st = tv.ProxSettings(10, 1e-300)
tv.tv_prox(img, 0.05, st)
torch.cuda.synchronize()
keep = []
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        tv.tv_prox(img, 0.05, st)
    e1.record()
    time.sleep(0.005)
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
    reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    w = next(iter(tv._ws_cache.values()))
    print(f"trial {trial:2d} {ms:7.3f} ms  sm {clk} MHz mem {mem} MHz reasons {reasons:#x} ws {w.data_ptr():#x}")
    keep.append(tv._ws_cache.copy())
    tv._ws_cache.clear()
