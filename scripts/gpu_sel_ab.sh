#!/bin/bash
# select A/B: parity tests of the candidate library (abl/libB.so), then same-box bench A/B
# of prebuilt product libraries abl/lib{A,B}.so on the select-heavy configs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/libB.so paper_2501_12162_b200/libadaserve.so
[ -n "$NO_TESTS" ] || timeout 900 python -m pytest tests -m gpu -q -x -k "${TESTK:-select or iteration or smoke}" --timeout 300 2>&1 | tail -3
for r in $(seq ${REPS:-2}); do for C in ${CONFIGS:-c3 c2}; do for v in ${LIBS:-A B}; do
  cp abl/lib$v.so paper_2501_12162_b200/libadaserve.so
  timeout 200 python bench.py --config $C --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C [$v] attn_us', round(r['attn_ms']*1e3,1), 'step_us', round(d['ms_per_step']*1e3,2), 'bd', d['breakdown_ms'].get('select'), d['breakdown_ms'].get('accept_commit'))"
done; done; done
