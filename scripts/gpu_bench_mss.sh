#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for C in ${CONFIGS:-c2}; do
timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/bench_mss_$C.json 2> gpurun_out/bench_mss_$C.err
tail -1 gpurun_out/bench_mss_$C.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$C', json.dumps(d['mss']))"
tail -3 gpurun_out/bench_mss_$C.err
done
