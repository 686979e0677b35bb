"""Randomised stress of as_beam_step against the oracle's beam_step (GPU; not
part of the test suite): random vocabularies (incl. sizes not a multiple of 4),
widths 1-16, batch sizes, peakedness and quantised (tied) probabilities; two
layers per case (layer 1 from the root, then w parents).
    python scripts/stress_beam.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2501_12162_b200 as ada  # noqa: E402
from tests.helpers import dev  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
for c in range(cases):
    V = int(rng.choice([5, 17, 1000, 4099, 8192, 65537, 128256]))
    width = int(rng.integers(1, min(16, V) + 1))
    n = int(rng.integers(1, max(2, min(300, int(4e7 // (V * width))))))
    d = 2
    stride = 1 + d * width
    par = np.zeros(n * stride, np.int32)
    prob = np.zeros(n * stride, np.float32)
    prob[::stride] = 1.0
    tok = np.zeros(n * stride, np.int32)
    g_par, g_prob, g_tok = dev(par), dev(prob), dev(tok)
    ties = rng.random() < 0.3
    ws = None
    for layer in (1, 2):
        w_in = 1 if layer == 1 else width
        z = rng.normal(0.0, float(rng.uniform(0.3, 6.0)), (n, w_in, V))
        e = np.exp(z - z.max(axis=-1, keepdims=True))
        P = (e / e.sum(axis=-1, keepdims=True)).astype(np.float32)
        if ties:
            P = (np.floor(P * 32.0) / 32.0).astype(np.float32)
        ws = ada.beam_step(layer, width, dev(P), g_par, g_prob, g_tok, stride, workspace=ws)
        base_prev = 0 if layer == 1 else 1
        base_new = 1 + (layer - 1) * width
        for i in range(n):
            fpar = prob[i * stride + base_prev: i * stride + base_prev + w_in]
            pr, tk, fv = oracle.beam_step(P[i], fpar, width)
            k = len(pr)
            o = i * stride + base_new
            par[o:o + k] = base_prev + pr
            tok[o:o + k] = tk
            prob[o:o + k] = fv
    ok = (ada.check_device_error(ws)[0] == 0 and np.array_equal(g_par.cpu().numpy(), par)
          and np.array_equal(g_tok.cpu().numpy(), tok)
          and np.array_equal(g_prob.cpu().numpy().view(np.int32), prob.view(np.int32)))
    if not ok:
        fails += 1
        print(f"FAIL case {c}: V={V} width={width} n={n} ties={ties}")
print(f"stress beam: {cases} cases x 2 layers, {fails} failures")
