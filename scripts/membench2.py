"""Per-SM TMA concurrency: 1 vs 2 vs 4 CTAs per SM (debug)."""
import ctypes, os, sys
os.environ.setdefault("AS_DEBUG_LIB", "1")  # debug build: experiment switches / instruments
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_12162_b200 as ada  # noqa: E402
L = ada.lib()
L.as_debug_stream_bw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
total = 1 << 30
buf = torch.randn(total // 2, dtype=torch.bfloat16, device="cuda")
sink = torch.zeros(8192, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def run(chunk, stages, mode, grid, reps=3):
    n = total // chunk
    order = torch.randperm(n, device="cuda").to(torch.int32)
    args = (buf.data_ptr(), order.data_ptr(), n, chunk, stages, mode, sink.data_ptr(), grid, st)
    assert L.as_debug_stream_bw(*args) == 0
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        L.as_debug_stream_bw(*args)
    e.record(); torch.cuda.synchronize()
    return total * reps / (s.elapsed_time(e) / 1e3) / 1e9
for chunk in (16384, 32768):
    for grid_mult in (1, 2, 3):
        for stages in (2, 3, 4):
            if stages * chunk * grid_mult > 200 * 1024:
                continue
            for mode in (3, 4):
                print(f"chunk {chunk//1024}KB CTAs/SM {grid_mult} stages {stages} issuers/CTA {1 if mode==3 else 2}: "
                      f"{run(chunk, stages, mode, 148 * grid_mult):6.0f} GB/s", flush=True)
