#!/bin/bash
# same-box A/B of two prebuilt product libraries (libadaserve_A.so vs libadaserve_B.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
P=paper_2501_12162_b200
for r in $(seq ${REPS:-2}); do for C in ${CONFIGS:-c2 c4 c5}; do for V in A B; do
  cp $P/libadaserve_$V.so $P/libadaserve.so
  timeout 200 python bench.py --config $C $EXTRA --steps 100 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C [$V] attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'step_us', round(d['ms_per_step']*1e3,1))"
done; done; done
cp $P/libadaserve_B.so $P/libadaserve.so
