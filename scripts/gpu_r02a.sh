#!/bin/bash
# r02 first check: full GPU suite + smoke + quick c2/c4 bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02a}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 300 > gpurun_out/tests_${TAG}.log 2>&1; grep -E "passed|failed|error" gpurun_out/tests_${TAG}.log | tail -5
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for C in c2 c4 c5; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --no-spec --no-e2e > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err
  tail -1 gpurun_out/bench_${TAG}_$C.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C', 'attn_ms', r['attn_ms'], r['bound'], r['achieved'], 'frac', r['frac'], 'step_ms', d['ms_per_step'], 'bd', d['breakdown_ms'])"
done
