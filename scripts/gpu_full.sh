#!/bin/bash
# Round evidence: all GPU tests, smoke, default bench (+ c3/c4/c5 lines), ncu launch list + full profile.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/tests_${TAG}.log 2>&1; grep -E "passed|failed" gpurun_out/tests_${TAG}.log | tail -2
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; tail -1 gpurun_out/bench_${TAG}_c2.json
for C in c3 c4 c5 c1; do
  timeout 400 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err; tail -1 gpurun_out/bench_${TAG}_$C.json | cut -c1-400
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
   --log-file gpurun_out/launches_${TAG}_c2.csv python bench.py --profile --steps 3 --warmup 3 --no-graph > /dev/null 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 2 -c 1 \
   -o gpurun_out/prof_attn_${TAG}_c2 -f python bench.py --profile --steps 1 --warmup 3 --no-graph > gpurun_out/ncu_attn_${TAG}.log 2>&1
echo "ncu attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 2 -c 1 \
   -o gpurun_out/prof_attn_${TAG}_c4 -f python bench.py --config c4 --profile --steps 1 --warmup 3 --no-graph > gpurun_out/ncu_attn_c4_${TAG}.log 2>&1
echo "ncu attn c4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"beam|argmax" -s 2 -c 3 \
   -o gpurun_out/prof_beam_${TAG}_c2 -f python bench.py --config c2 --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > gpurun_out/ncu_beam_${TAG}.log 2>&1
echo "ncu beam rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_trees|walk_commit" -s 4 -c 2 \
   -o gpurun_out/prof_small_${TAG}_c2 -f python bench.py --profile --steps 2 --warmup 3 --no-graph > gpurun_out/ncu_small_${TAG}.log 2>&1
echo "ncu small rc=$?"
for W in 8; do for C in c2 c4 c5; do
  AS_BENCH_EMULATE_WORLD=$W timeout 300 python bench.py --config $C --no-cpu-baseline --no-spec > gpurun_out/bench_${TAG}_${C}_w$W.json 2>/dev/null
  echo "emulated w$W $C rc=$?"
done; done
