#!/bin/bash
# FMA-pipe share of the NQ=2 softmax exponentials: abl/libP{8,4,2}.so (one pair in 8 / 4 / 2) vs libW (none)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/libP4.so paper_2501_12162_b200/libadaserve.so
timeout 1200 python -m pytest tests -m gpu -q -k "attn or smoke or iteration" --timeout 300 > gpurun_out/tests_poly.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/tests_poly.log | tail -6
NO_TESTS=1 REPS=2 CONFIGS="c4 c5" LIBS="W P8 P4 P2" bash scripts/gpu_sel_ab.sh 2>&1 | grep "\["
