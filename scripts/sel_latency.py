"""Latency profile of the select kernel: per-launch time of a CUDA graph of
back-to-back launches, for each AS_SEL_STOP value (the kernel returns after
phase k; debug only).  Usage: python scripts/sel_latency.py c2"""
import os
os.environ.setdefault("AS_DEBUG_LIB", "1")  # debug build: experiment switches / instruments
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 2:  # child: one stop value
    import numpy as np
    import torch
    import bench
    W = bench.make_workload(sys.argv[1], "cuda")
    reps = 50
    for _ in range(3):
        bench.run_select(W)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            bench.run_select(W)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e3 / reps)
    print(f"{sys.argv[1]} stop={sys.argv[2]} pdl={os.environ.get('AS_PDL', '1')}: {best:.2f} us/launch")
else:
    for pdl in os.environ.get("SEL_PDL", "1 0").split():
        for stop in os.environ.get("SEL_STOPS", "0 1 2 3 4 5 6 99").split():
            env = dict(os.environ, AS_SEL_STOP=stop, AS_PDL=pdl)
            r = subprocess.run([sys.executable, __file__, sys.argv[1], stop], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-500:])
