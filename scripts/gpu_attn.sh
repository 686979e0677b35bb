#!/bin/bash
# attention iteration: build, attention parity tests, c2/c4/c5 bench lines (+ optional ncu of one config)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "attn or umma" --timeout 120 > gpurun_out/tests_attn_${TAG}.log 2>&1; grep -E "passed|failed|error|Error" gpurun_out/tests_attn_${TAG}.log | tail -8
for C in ${CONFIGS:-c2 c4 c5}; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --no-spec --no-e2e > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err
  tail -1 gpurun_out/bench_${TAG}_$C.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C', 'attn_ms', r['attn_ms'], r['bound'], r['achieved'], 'frac', r['frac'], 'hbm_frac', r['hbm_frac'], 'step_ms', d['ms_per_step'], 'bd', d['breakdown_ms'])" || tail -5 gpurun_out/bench_${TAG}_$C.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 2 -c 1 \
     -o gpurun_out/prof_attn_${TAG}_$NCU -f python bench.py --config $NCU --profile --steps 1 --warmup 3 --no-graph > gpurun_out/ncu_${TAG}_$NCU.log 2>&1
  echo "ncu rc=$?"
fi
