#!/bin/bash
# same-box A/B of a debug-build environment switch: ENVA vs ENVB, alternating, REPS times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
export AS_DEBUG_LIB=1
for r in $(seq ${REPS:-2}); do for C in ${CONFIGS:-c2 c4 c5}; do for E in "$ENVA" "$ENVB"; do
  env $E timeout 200 python bench.py --config $C $EXTRA --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C [$E] attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'])"
done; done; done
