#!/bin/bash
# beam scan through an LDGSTS ring (abl/libB3.so: 3 stages, libB2: 2) vs HEAD (libH): parity + same-box A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp abl/lib${TESTLIB:-B3}.so paper_2501_12162_b200/libadaserve.so
timeout 900 python -m pytest tests -m gpu -q -k "beam or smoke" --timeout 300 > gpurun_out/tests_beam.log 2>&1; grep -E "passed|failed|FAILED" gpurun_out/tests_beam.log | tail -6
for r in 1 2; do for C in c2 c3 c5; do for v in ${LIBS:-H B3 B2}; do
  cp abl/lib$v.so paper_2501_12162_b200/libadaserve.so
  timeout 300 python bench.py --config $C --steps 50 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['speculation']
print('$C [$v] beam layer_us', s['layer_us'], 'hbm_frac', s['hbm_frac'])"
done; done; done
