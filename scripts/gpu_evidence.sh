#!/bin/bash
# Round evidence: GPU tests, smoke, bench lines (c2 default + c1/c3/c3b/c4/c5), launch list, ncu of
# the attention (c2, c4) and MSS kernels, compute-sanitizer on smoke().  TAG names the files.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/tests_${TAG}.log 2>&1; grep -E "passed|failed" gpurun_out/tests_${TAG}.log | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
fi
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; tail -1 gpurun_out/bench_${TAG}_c2.json | cut -c1-300
for C in ${CONFIGS:-c1 c3 c3b c4 c5}; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err
  tail -1 gpurun_out/bench_${TAG}_$C.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C', 'value', d['value'], 'attn_us', round(r['attn_ms']*1e3,1), r['bound'], 'frac', r['frac'], 'hbm_frac', r['hbm_frac'], 'step_us', round(d['ms_per_step']*1e3,1), 'bd', d['breakdown_ms'])" 2>&1 | tail -1
done
if [ -z "$SKIP_NCU" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_${TAG}_c2.csv python bench.py --profile --steps 3 --warmup 3 --no-graph > /dev/null 2>&1
echo "launches rc=$?"
for C in c2 c4; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 2 -c 1 \
   -o gpurun_out/prof_attn_${TAG}_$C -f python bench.py --config $C --profile --steps 1 --warmup 3 --no-graph > gpurun_out/ncu_attn_${TAG}_$C.log 2>&1
echo "ncu attn $C rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_trees|walk_commit" -s 4 -c 2 \
   -o gpurun_out/prof_small_${TAG}_c2 -f python bench.py --profile --steps 2 --warmup 3 --no-graph > gpurun_out/ncu_small_${TAG}.log 2>&1
echo "ncu small rc=$?"
fi
if [ -z "$SKIP_SHARDS" ]; then
for W in 2 4 8; do for C in c2 c4 c5; do
  AS_BENCH_EMULATE_WORLD=$W timeout 300 python bench.py --config $C --no-cpu-baseline --no-spec --no-e2e > gpurun_out/bench_${TAG}_${C}_w$W.json 2>/dev/null
  tail -1 gpurun_out/bench_${TAG}_${C}_w$W.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C w$W attn_us', round(r['attn_ms']*1e3,1), 'step_us', round(d['ms_per_step']*1e3,1))" 2>&1 | tail -1
done; done
fi
if [ -z "$SKIP_SEL" ]; then
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
for C in c2 c3 c4; do AS_DEBUG_LIB=1 SEL_PDL=1 SEL_STOPS="99" timeout 300 python scripts/sel_latency.py $C 2>&1 | tail -1; done
fi
if [ -z "$SKIP_SAN" ]; then
for TOOL in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${TOOL}_${TAG}.log 2>&1
  echo "sanitizer $TOOL rc=$?"; grep -E "ERROR SUMMARY|smoke ok" gpurun_out/sanitizer_${TOOL}_${TAG}.log | tail -2
done
fi
