#!/bin/bash
# Iteration run: build, selected GPU tests (TESTK=pytest -k expr, empty = skip),
# bench lines for CFGS, optional ncu of the small kernels (NCU_SMALL=1) or the
# attention kernel (NCU_ATTN=cfg).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail -20 gpurun_out/build_${TAG}.log; exit 1; }
if [ -n "$TESTK" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$TESTK" > gpurun_out/tests_${TAG}.log 2>&1
  echo "tests rc=$?"; tail -4 gpurun_out/tests_${TAG}.log
fi
for C in ${CFGS:-c2}; do
  timeout 400 python bench.py --config $C --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err
  echo "bench $C rc=$?"; tail -1 gpurun_out/bench_${TAG}_$C.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C', 'step_ms', d['ms_per_step'], 'tok/s %.3g' % d['value'], 'attn_ms', r['attn_ms'], 'bound', r['bound'], 'frac', r['frac'], 'hbm', r['hbm_frac'], 'tc_burst', r['tensor_frac_burst'], 'bd', d['breakdown_ms'], 'e2e', (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1
  tail -3 gpurun_out/bench_${TAG}_$C.err
done
if [ -n "$NCU_SMALL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_trees|walk_commit" -s 4 -c 2 \
     -o gpurun_out/prof_small_${TAG} -f python bench.py --config ${NCU_SMALL} --profile --steps 2 --warmup 3 --no-graph > gpurun_out/ncu_small_${TAG}.log 2>&1
  echo "ncu small rc=$?"
fi
if [ -n "$NCU_ATTN" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 2 -c 1 \
     -o gpurun_out/prof_attn_${TAG}_${NCU_ATTN} -f python bench.py --config ${NCU_ATTN} --profile --steps 1 --warmup 3 --no-graph > gpurun_out/ncu_attn_${TAG}.log 2>&1
  echo "ncu attn rc=$?"
fi
if [ -n "$LAUNCHES" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
     --log-file gpurun_out/launches_${TAG}_${LAUNCHES}.csv python bench.py --config $LAUNCHES --profile --steps 3 --warmup 3 --no-graph > /dev/null 2>&1
  echo "launches rc=$?"
fi
