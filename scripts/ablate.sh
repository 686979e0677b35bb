#!/bin/bash
# Incremental in-step cost of each kernel: step time with one call skipped (ablation, debug only).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1 AS_DEBUG_LIB=1  # debug build (experiment switches)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for C in ${CFGS:-c2}; do
  for SK in none select accept attention "select,accept"; do
    AS_BENCH_SKIP=$SK timeout 300 python bench.py --config $C --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$C skip=$SK step_us %.1f' % (d['ms_per_step']*1e3))"
  done
done
