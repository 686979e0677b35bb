#!/bin/bash
# bench (graph) + ncu launch list + ncu --set full of the attention kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CFG=${CFG:-c2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err
tail -2 gpurun_out/bench_${TAG}_${CFG}.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_${TAG}_${CFG}.csv python bench.py --config $CFG --profile --steps 3 --warmup 3 --no-graph > /dev/null 2>&1
echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn_tc -s 2 -c 1 \
   -o gpurun_out/prof_attn_${TAG}_${CFG} -f python bench.py --config $CFG --profile --steps 1 --warmup 3 --no-graph > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_${TAG}.log
