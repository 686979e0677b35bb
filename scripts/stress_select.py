"""Randomised stress of as_select_trees against the oracle's literal Alg. 2
(GPU; not part of the test suite): the fuzz recipe of tests/test_select_fuzz
with fresh seeds, more iterations and a wider size mix (1-4096 requests, up to
257 candidates each, forced f-hat ties, repeated A values).
    python scripts/stress_select.py [iterations] [seed]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from tests.test_gpu_parity import _assert_select_equal, _gpu_select  # noqa: E402
import paper_2501_12162_b200 as ada  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
fails = 0
for it in range(iters):
    kind = it % 5
    n = int(rng.integers(1, [10, 80, 500, 2000, 4097][kind]))
    maxn = int([257, 60, 40, 12, 5][kind])  # <= 1 + AS_MAX_CAND (more is a flagged precondition error)
    F = synth.random_forest(rng, n, maxn, tie_prob=float(rng.choice([0.0, 0.3, 0.8])))
    N = int(F["cand_offsets"][-1])
    F["cand_token"] = rng.integers(0, 128256, N).astype(np.int32)
    A = rng.uniform(-1, 9, n)
    if rng.random() < 0.5:
        A[rng.integers(0, n, max(1, n // 3))] = A[0]
    d = int(rng.integers(0, 10))
    n_max = int(rng.integers(0, 300))
    B = int(rng.integers(n, N + 5))
    try:
        got = _gpu_select(ada, F, A, d, n_max, B)
        _assert_select_equal(F, A, d, n_max, B, got)
    except AssertionError as e:
        fails += 1
        print(f"FAIL it={it} n={n} N={N} d={d} n_max={n_max} B={B}: {str(e)[:200]}")
print(f"stress select: {iters} forests, {fails} failures")
