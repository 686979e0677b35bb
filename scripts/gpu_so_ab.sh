#!/bin/bash
# same-box A/B of prebuilt product libraries abl/lib{A,B,...}.so (built locally from two code versions)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in $(seq ${REPS:-2}); do for C in ${CONFIGS:-c2 c4}; do for v in ${LIBS:-A B}; do
  cp abl/lib$v.so paper_2501_12162_b200/libadaserve.so
  timeout 200 python bench.py --config $C $EXTRA --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C [$v] attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'step_us', round(d['ms_per_step']*1e3,1))"
done; done; done
