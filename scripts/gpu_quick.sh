#!/bin/bash
# selftests one by one (each under its own timeout), attention parity, short bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in $(python -m pytest tests/test_gpu_parity.py --collect-only -q -k umma 2>/dev/null | grep "::"); do
  timeout 60 python -m pytest "$t" -q 2>&1 | tail -1 | sed "s|^|$t: |"
done
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "attn" 2>&1 | tail -5
for SK in 0 1; do
timeout 200 python bench.py --schedule split=$SK --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('c2 streamk=$SK', 'attn_ms', r['attn_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], 'step_ms', d['ms_per_step'], 'bd', d['breakdown_ms'])"
done
