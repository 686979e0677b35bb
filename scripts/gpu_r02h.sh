#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in B R; do
  cp abl/lib$v.so paper_2501_12162_b200/libadaserve.so
  echo "== full-size attention tests, lib $v"
  timeout 900 python -m pytest tests -m gpu -q -k "full_size_sampled" --timeout 300 2>&1 | grep -E "passed|failed|FAILED" | tail -8
done
cp abl/libB.so paper_2501_12162_b200/libadaserve.so
echo "== select tests, lib B"
timeout 900 python -m pytest tests -m gpu -q -k "select" --timeout 300 2>&1 | grep -E "passed|failed|FAILED" | tail -5
NO_TESTS=1 REPS=2 CONFIGS="c3 c2" LIBS="A B" bash scripts/gpu_sel_ab.sh 2>&1 | grep -v "^$" | grep "\[" 
REPS=1 WORLDS=8 CONFIGS="c2 c4 c5" LIBS="B S2 S3" bash scripts/gpu_shard_ab.sh
