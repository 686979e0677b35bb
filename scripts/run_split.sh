cd "${GRAFT_REPO_ROOT:-/root/repo}"
export TAG=sp2 TESTK="attn or iteration" CFGS="c2 c4 c5"
bash scripts/gpu_iter.sh
for W in 4 8; do for C in c2 c4 c5; do
  AS_BENCH_EMULATE_WORLD=$W timeout 300 python bench.py --config $C --steps 20 --warmup 5 --no-cpu-baseline --no-spec > gpurun_out/bench_sp2_${C}_w$W.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bench_sp2_${C}_w$W.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$C w$W attn_ms', r['attn_ms'], 'step', d['ms_per_step'])"
done; done
AS_BENCH_EMULATE_WORLD=8 timeout 200 python scripts/attn_trace.py --config c2 > gpurun_out/trace_sp2.txt 2>&1; tail -8 gpurun_out/trace_sp2.txt
