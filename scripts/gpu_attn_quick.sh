#!/bin/bash
# attention parity tests + c2..c5 attention timings of the current product build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "${TESTK:-attn}" --timeout 300 2>&1 | tail -3
for r in $(seq ${REPS:-1}); do for C in ${CONFIGS:-c2 c3 c4 c5}; do
timeout 200 python bench.py --config $C $EXTRA --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C attn_us', round(r['attn_ms']*1e3,1), r['bound'], 'frac', r['frac'], 'step_us', round(d['ms_per_step']*1e3,1), 'value', d['value'])"
done; done
