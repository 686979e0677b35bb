#!/bin/bash
# softmax exponentials-first (abl/libE.so) vs warpgroup roles only (libW) vs the committed build (libF)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/libE.so paper_2501_12162_b200/libadaserve.so
timeout 1200 python -m pytest tests -m gpu -q -k "attn or smoke or iteration" --timeout 300 > gpurun_out/tests_ef.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/tests_ef.log | tail -6
NO_TESTS=1 REPS=2 CONFIGS="c4 c5" LIBS="F W E" bash scripts/gpu_sel_ab.sh 2>&1 | grep "\["
NO_TESTS=1 REPS=1 CONFIGS="c2 c3" LIBS="F E" bash scripts/gpu_sel_ab.sh 2>&1 | grep "\["
