#!/bin/bash
# attention plan with fewer barriers (abl/libX.so) vs HEAD (abl/libH.so): parity, same-box A/B, plan trace
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/libX.so paper_2501_12162_b200/libadaserve.so
timeout 1200 python -m pytest tests -m gpu -q -k "attn or smoke or iteration or dist" --timeout 300 > gpurun_out/tests_plan.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/tests_plan.log | tail -6
NO_TESTS=1 REPS=2 CONFIGS="c2 c3 c4" LIBS="H X" bash scripts/gpu_sel_ab.sh 2>&1 | grep "\["
REPS=2 WORLDS=8 CONFIGS="c2" LIBS="H X" bash scripts/gpu_shard_ab.sh 2>&1
AS_ATTN_DEBUG_MODE=6 CFGS="c2" WORLDS="1" bash scripts/run_trace.sh 2>&1 | grep -E "per CTA|plan done"
