"""Run bench.py's multi-GPU arm (run_multi: row slabs, NCCL) with whatever world size
torchrun gives it -- including 1, to exercise the NCCL plumbing on a single GPU:
    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 \\
        --master-port 29511 tools/bench_dist_check.py --steps 10 --warmup 3"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
bench.run_multi(ap.parse_args())
