#!/bin/bash
# per-rank shard A/B (AS_BENCH_EMULATE_WORLD): prebuilt libraries abl/lib{LIBS}.so, same box
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in $(seq ${REPS:-2}); do for W in ${WORLDS:-8 4}; do for C in ${CONFIGS:-c2 c4 c5}; do for v in ${LIBS:-B S2 S3}; do
  cp abl/lib$v.so paper_2501_12162_b200/libadaserve.so
  AS_BENCH_EMULATE_WORLD=$W timeout 200 python bench.py --config $C --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C w$W [$v] attn_us', round(r['attn_ms']*1e3,1), 'hbm_frac', r.get('hbm_frac'), 'step_us', round(d['ms_per_step']*1e3,2))"
done; done; done; done
