#!/bin/bash
# attention time under the debug modes (0 full, 1 no softmax math, 2 no MMA either) for shape overrides
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1 AS_DEBUG_LIB=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
for C in ${CONFIGS:-c4}; do for SH in ${SHAPES:-"NQ=2" "CS=2"}; do for M in 0 1 2; do
  AS_ATTN_DEBUG_MODE=$M timeout 120 python bench.py --config $C --schedule "$(echo ${SH} | tr A-Z a-z)" --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C $SH mode $M attn_us', round(r['attn_ms']*1e3,1))"
done; done; done
