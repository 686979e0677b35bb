"""Randomised stress of the bf16 attention path against the oracle (GPU; not
part of the test suite): random batch sizes, tree sizes/shapes, prefix lengths
(incl. 0 and page-boundary values), head layouts and head dims, under every
schedule switch (nq 1/2, split 0/1 via as_tree_verify_attn_sched).  Usage:
    python scripts/stress_attn.py [cases] [seed]
Prints one line per failing case and a summary."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from tests.helpers import oracle_attn, workload_to_device  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(seed)
import paper_2501_12162_b200 as ada  # noqa: E402

worst, fails = 0.0, 0
for c in range(cases):
    n = int(rng.choice([1, 2, 3, 7, 20, 64, 150]))
    n_q, n_kv = [(32, 8), (64, 8), (8, 8), (16, 2), (32, 4), (4, 1)][int(rng.integers(0, 6))]
    G = n_q // n_kv
    d = int(rng.choice([64, 128]))
    kmax = min(128, max(1, 512 // G))
    sizes = rng.integers(1, kmax + 1, n)
    kv = rng.integers(0, 3000, n)
    kv[rng.random(n) < 0.2] = 0
    edge = rng.random(n) < 0.2
    kv[edge] = 64 * rng.integers(0, 40, int(edge.sum()))
    while float((sizes * (kv + sizes)).sum()) * n_q * d > 3e9:  # keep the fp64 oracle to seconds
        kv = kv // 2
        sizes = np.maximum(1, sizes * 3 // 4)
    shape = str(rng.choice(["random", "chain", "star"]))
    w = synth.tree_workload(rng, sizes, kv, n_q, n_kv, d, 64, shape=shape, bf16=True)
    scale = np.float32(1.0 / np.sqrt(d))
    ref, ref_lse = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    for nq in ("1", "2"):
        for sk in ("0", "1"):
            ws = ada.Workspace(256)
            out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"],
                                            g["page_table"], g["kv_len"], g["tree_offsets"], g["tree_parent"],
                                            scale, want_lse=True, workspace=ws, schedule=f"nq={nq},split={sk}")
            code = ada.check_device_error(ws)[0]
            err = float(np.abs(out.float().cpu().numpy() - ref).max())
            lerr = float(np.abs(lse.cpu().numpy() - ref_lse).max())
            worst = max(worst, err)
            if code != 0 or not (err <= 2e-2) or not (lerr <= 2e-2):
                fails += 1
                print(f"FAIL case {c} nq={nq} sk={sk}: n={n} heads={n_q}/{n_kv} d={d} shape={shape} "
                      f"sizes[:5]={sizes[:5].tolist()} kv[:5]={kv[:5].tolist()} err={err:.3g} lse={lerr:.3g} code={code}")
print(f"stress: {cases} cases x 4 schedules, {fails} failures, worst max-abs {worst:.3g}")
