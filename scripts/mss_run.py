"""Run as_mss_verify on the bench's c2 MSS inputs (for ncu / timing experiments).
    python scripts/mss_run.py [--mode walk|all] [--iters N] [--config c2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="walk")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--config", default="c2")
a = ap.parse_args()
torch.cuda.set_device(0)
W = bench.make_workload(a.config, "cuda")
os.environ["AS_MSS_ONLY_MODE"] = a.mode
r = bench.measure_mss(W, a.iters)
print(r)
