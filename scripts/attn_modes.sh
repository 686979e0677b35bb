#!/bin/bash
# Timing experiments for the bf16 attention kernel (debug modes produce wrong outputs).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1 AS_DEBUG_LIB=1  # debug build (experiment switches)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
one() {
  timeout 200 python bench.py --config $CFG --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$CFG mode=${AS_ATTN_DEBUG_MODE:-0} contig=${AS_BENCH_CONTIGUOUS_PAGES:-0}', 'attn_ms', r['attn_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], 'step_ms', d['ms_per_step'], 'bd', d['breakdown_ms'], 'clk', d['clocks'])"
}
for CFG in ${CFGS:-c2}; do
  for M in ${MODES:-0 2}; do AS_ATTN_DEBUG_MODE=$M one; done
done
