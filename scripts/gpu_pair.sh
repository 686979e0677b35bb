#!/bin/bash
# CTA-pair attention first light: one small case under a hard timeout, then the rest
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 60 python -m pytest "tests/test_gpu_parity.py::test_attn_bf16_cta_pair[1-4]" -q -x --timeout 40 2>&1 | tail -4
rc=${PIPESTATUS[0]}; echo "first rc=$rc"; [ $rc -ne 0 ] && exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "cta_pair" --timeout 60 2>&1 | tail -4
for C in c4 c5; do for SH in auto "pair=1"; do
  S=""; [ "$SH" != "auto" ] && S="--schedule $SH"
  timeout 120 python bench.py --config $C $S --steps 50 --no-cpu-baseline --no-spec --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$C $SH attn_us', round(r['attn_ms']*1e3,1), 'frac', r['frac'], 'hbm_frac', r['hbm_frac'])"
done; done
