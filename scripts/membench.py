"""HBM streaming micro-benchmark (as_debug_stream_bw) -- sizing the attention load path."""
import ctypes
import os
os.environ.setdefault("AS_DEBUG_LIB", "1")  # debug build: experiment switches / instruments
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_12162_b200 as ada  # noqa: E402

L = ada.lib()
L.as_debug_stream_bw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
total = 1 << 30  # 1 GiB
buf = torch.randn(total // 2, dtype=torch.bfloat16, device="cuda")
sink = torch.zeros(4096, dtype=torch.int64, device="cuda")
nsm = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream().cuda_stream


def run(chunk, stages, mode, rand, grid=nsm, reps=3):
    n = total // chunk
    order = (torch.randperm(n, device="cuda") if rand else torch.arange(n, device="cuda")).to(torch.int32)
    args = (buf.data_ptr(), order.data_ptr(), n, chunk, stages, mode, sink.data_ptr(), grid, st)
    assert L.as_debug_stream_bw(*args) == 0
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        L.as_debug_stream_bw(*args)
    e.record()
    torch.cuda.synchronize()
    return total * reps / (s.elapsed_time(e) / 1e3) / 1e9


print("SMs", nsm)
for mode in (3, 4, 5, 6):
    for chunk in (16384, 32768):
        for stages in (4, 8, 12):
            if stages * chunk > 200 * 1024:
                continue
            r = [run(chunk, stages, mode, rand) for rand in (False, True)]
            print(f"mode {mode} chunk {chunk // 1024:2d}KB stages {stages:2d} ({stages * chunk // 1024:3d}KB in flight): "
                  f"seq {r[0]:6.0f} GB/s  random {r[1]:6.0f} GB/s")
print("modes: 3 tensor-1thr 4 tensor-2thr 5 tensor-4thr 6 tensor-8thr")
