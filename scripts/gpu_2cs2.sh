#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 120 python -m pytest "tests/test_gpu_parity.py::test_attn_bf16[2cs2-1]" -q -x --timeout 60 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "2cs2" --timeout 200 2>&1 | tail -3
for C in c4 c5; do for SH in "nq=2" "nq=2,cs=2"; do
  timeout 120 python bench.py --config $C --schedule "$SH" --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C $SH attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'hbm_frac', r['hbm_frac'])"
done; done
