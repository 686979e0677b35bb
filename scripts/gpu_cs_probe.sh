#!/bin/bash
# first light of the cluster (multicast) attention shapes: one small case each, hard timeouts
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for t in "test_attn_bf16[cs2-1]" "test_attn_bf16[cs4-1]" "test_attn_bf16[cs2-5]"; do
  timeout 90 python -m pytest "tests/test_gpu_parity.py::$t" -q -x --timeout 60 2>&1 | tail -2
  rc=${PIPESTATUS[0]}; echo "$t rc=$rc"; if [ $rc -ne 0 ]; then exit 1; fi
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "attn" --timeout 120 > gpurun_out/tests_cs.log 2>&1; grep -E "passed|failed|Error" gpurun_out/tests_cs.log | tail -5
for CS in 2 4; do for C in c4 c5; do
  timeout 120 python bench.py --config $C --schedule cs=$CS --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('cs$CS $C', 'attn_ms', r['attn_ms'], r['bound'], r['achieved'], 'frac', r['frac'], 'hbm_frac', r['hbm_frac'], 'step_ms', d['ms_per_step'])"
done; done
