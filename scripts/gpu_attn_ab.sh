#!/bin/bash
# attention parity subset + bench lines per schedule (A/B)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "${TESTS:-attn}" --timeout 300 2>&1 | tail -3
fi
for C in ${CONFIGS:-c2 c4 c5}; do for SH in ${SCHEDS:-auto}; do
  S=""; [ "$SH" != "auto" ] && S="--schedule $SH"
  timeout 200 python bench.py --config $C $S --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C $SH attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'hbm_frac', r['hbm_frac'], 'step_us', round(d['ms_per_step']*1e3,1), 'p10/p90', d['distribution_ms']['attention']['p10'], d['distribution_ms']['attention']['p90'])"
done; done
