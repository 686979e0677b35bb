#!/bin/bash
# same-box A/B of PRODUCT builds that differ in compile-time defines: VARIANTS="name:defines;..."
# e.g. VARIANTS="p0:-DAS_POLY_COLS=0;p2:-DAS_POLY_COLS=2"; each built once, swapped in per run
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p /tmp/libab
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  n=${v%%:*}; d=${v#*:}
  AS_NVCC_DEFINES="$d" python -m paper_2501_12162_b200.build --force > /dev/null 2>&1 || { echo "build $n failed"; exit 1; }
  cp paper_2501_12162_b200/libadaserve.so /tmp/libab/$n.so
done
for r in $(seq ${REPS:-2}); do for C in ${CONFIGS:-c4 c5}; do for v in "${VS[@]}"; do
  n=${v%%:*}
  cp /tmp/libab/$n.so paper_2501_12162_b200/libadaserve.so
  timeout 200 python bench.py --config $C $EXTRA --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C [$n] attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'step_us', round(d['ms_per_step']*1e3,1))"
done; done; done
