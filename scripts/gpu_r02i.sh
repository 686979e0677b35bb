#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/libF.so paper_2501_12162_b200/libadaserve.so
echo "== all GPU tests, lib F"
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/tests_r02i_F.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/tests_r02i_F.log | tail -8
NO_TESTS=1 REPS=2 CONFIGS="c2 c4 c5" LIBS="R F" bash scripts/gpu_sel_ab.sh 2>&1 | grep "\["
