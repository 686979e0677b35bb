#!/bin/bash
# tail stream-K merge A/B: attention parity, then c2 balanced (TAIL=1) vs forced tail (TAIL=2), c3/c4 default
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "attn" --timeout 300 2>&1 | tail -3
CONFIGS="${CONFIGS:-c2}" ENVA="AS_ATTN_TAIL=1" ENVB="AS_ATTN_TAIL=2" REPS=${REPS:-3} bash scripts/gpu_ab_env.sh
for C in c3 c4 c5; do
timeout 200 python bench.py --config $C --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C default attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'])"
done
