#!/bin/bash
# A/B matrix for the bf16 attention kernel on one box (with a TMA streaming calibration).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1 AS_DEBUG_LIB=1  # debug build (experiment switches)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python - <<'PY'
import ctypes, torch, sys
sys.path.insert(0, '.')
import paper_2501_12162_b200 as ada
L = ada.lib()
L.as_debug_stream_bw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
total = 1 << 30
buf = torch.randn(total // 2, dtype=torch.bfloat16, device="cuda")
sink = torch.zeros(4096, dtype=torch.int64, device="cuda")
for chunk, mode in ((16384, 4), (32768, 3)):
    n = total // chunk
    order = torch.randperm(n, device="cuda").to(torch.int32)
    args = (buf.data_ptr(), order.data_ptr(), n, chunk, 4, mode, sink.data_ptr(), 148, torch.cuda.current_stream().cuda_stream)
    L.as_debug_stream_bw(*args); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); [L.as_debug_stream_bw(*args) for _ in range(3)]; e.record(); torch.cuda.synchronize()
    print(f"calib TMA {chunk//1024}KB x{2 if mode==4 else 1}thr: {3*total/(s.elapsed_time(e)/1e3)/1e9:.0f} GB/s")
a = torch.empty(1 << 29, dtype=torch.bfloat16, device="cuda"); b = torch.empty_like(a)
b.copy_(a); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); [b.copy_(a) for _ in range(5)]; e.record(); torch.cuda.synchronize()
print(f"calib copy: {5*2*a.numel()*2/(s.elapsed_time(e)/1e3)/1e9:.0f} GB/s")
PY
one() {
  timeout 200 python bench.py --config ${CFG:-c2} --schedule "$SCHED" --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('${CFG:-c2} $TAG', 'attn_ms', r['attn_ms'], 'GB/s', r['achieved'], 'frac', r['frac'], 'step_ms', d['ms_per_step'], 'bd', d['breakdown_ms'])"
}
for CFG in ${CFGS:-c2}; do
for KL in 1 2 3; do
TAG="klead$KL" AS_ATTN_KLEAD=$KL one
done
TAG="mode2" AS_ATTN_DEBUG_MODE=2 one
TAG="streamk0" SCHED="split=0" one
done
