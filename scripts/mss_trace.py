"""Per-node timeline of the MSS walk kernel, cluster 0 (debug build).
    AS_DEBUG_LIB=1 python scripts/mss_trace.py [--config c2]
Events (globaltimer ns, relative to the first node start): 0 node start,
1 rows landed, 2 first mass pass done, 3 decisions done, 5 bonus done;
4 = rejections, 6 = node id, 7 = children."""
import argparse
import os
os.environ.setdefault("AS_DEBUG_LIB", "1")
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_12162_b200 as ada  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
args = ap.parse_args()
W = bench.make_workload(args.config, "cuda")
ws = ada.Workspace(256 + 64 * 64 + 4096, "cuda")
W["mss_ws"] = ws
bench.measure_mss(W, 3)
t = ws.view[256:256 + 64 * 64].view(torch.int64).cpu().numpy().reshape(64, 8)
t0 = t[0, 0]
for k in range(32):
    if t[k, 0] == 0:
        break
    r = t[k]
    rel = lambda e: (r[e] - t0) / 1e3 if r[e] else float("nan")
    print(f"node {r[6]:3d} kids {r[7]:2d} rej {r[4]:2d} | start {rel(0):7.2f} loaded {rel(1):7.2f} "
          f"pass0 {rel(2):7.2f} decided {rel(3):7.2f} bonus {rel(5):7.2f} us")
    if k < 16 and r[4] > 0:
        a, b = t[32 + k], t[48 + k]
        print("   rejection passes (start, pass done):", [(round((a[j] - t0) / 1e3, 2), round((b[j] - t0) / 1e3, 2))
                                                     for j in range(min(8, r[4]))])
