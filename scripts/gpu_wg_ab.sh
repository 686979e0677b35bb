#!/bin/bash
# warpgroup-aligned roles + setmaxnreg (abl/libW.so) vs the committed build (abl/libF.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/libW.so paper_2501_12162_b200/libadaserve.so
timeout 1200 python -m pytest tests -m gpu -q -k "attn or smoke or iteration" --timeout 300 > gpurun_out/tests_wg.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/tests_wg.log | tail -6
NO_TESTS=1 REPS=2 CONFIGS="c4 c5" LIBS="F W" bash scripts/gpu_sel_ab.sh 2>&1 | grep "\["
