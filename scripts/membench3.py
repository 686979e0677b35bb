"""TMA streaming rate vs CTAs/SM, ring depth and issuing threads (debug)."""
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
chunk = 16384
for cps, stage_list in ((1, (2, 4, 6, 8, 12)), (2, (2, 3, 4, 5, 6)), (3, (2, 3, 4))):
    for stages in stage_list:
        res = []
        for mode in (0, 1, 5, 3):
            if {0: 1, 1: 2, 5: 4, 3: 1}[mode] > stages:
                continue
            res.append(f"m{mode} {run(chunk, stages, mode, 148 * cps):5.0f}")
        print(f"16KB CTAs/SM {cps} stages {stages}: " + "  ".join(res), flush=True)
