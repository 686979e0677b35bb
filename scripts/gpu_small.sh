#!/bin/bash
# GPU tests + c2 bench + ncu --set full of the small kernels (select, accept).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
CFG=${CFG:-c2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
[ -n "$TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err
tail -1 gpurun_out/bench_${TAG}_${CFG}.json | cut -c1-300; tail -1 gpurun_out/bench_${TAG}_${CFG}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['breakdown_ms'], d['roofline']['frac'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_trees|walk_commit" -s 4 -c 2 \
   -o gpurun_out/prof_small_${TAG}_${CFG} -f python bench.py --config $CFG --profile --steps 2 --warmup 3 --no-graph > gpurun_out/ncu_small_${TAG}.log 2>&1
echo "ncu small rc=$?"
