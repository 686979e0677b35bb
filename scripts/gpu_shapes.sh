#!/bin/bash
# attention CTA-shape probe (results identical; schedule only): c4/c5 under NQ=1, NQ=2, CS=2, CS=4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for C in ${CONFIGS:-c4 c5}; do for SH in ${SHAPES:-"NQ=1" "NQ=2" "CS=2" "CS=4"}; do
  timeout 120 python bench.py --config $C --schedule "$(echo ${SH} | tr A-Z a-z)" --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C $SH attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'hbm_frac', r['hbm_frac'], 'step_us', round(d['ms_per_step']*1e3,1))"
done; done
