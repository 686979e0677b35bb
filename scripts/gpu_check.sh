#!/bin/bash
# One gpurun pass: device info, GPU parity tests (each group under its own
# timeout so a hung kernel cannot eat the budget), a short bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nvidia-smi; nproc; lscpu | head -20; } > gpurun_out/device.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { local name=$1; local t=$2; shift 2; echo "== $name" ; timeout $t "$@" > gpurun_out/$name.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/$name.log; }
run umma 180 python -m pytest tests/test_gpu_parity.py -k umma -q
run select_accept 300 python -m pytest tests/test_gpu_parity.py -k "select or accept" -q
run attn_fp32 300 python -m pytest tests/test_gpu_parity.py -k attn_fp32 -q
run attn_bf16 300 python -m pytest tests/test_gpu_parity.py -k "attn_bf16 and not full" -q
run attn_full 400 python -m pytest tests/test_gpu_parity.py -k "full" -q
run smoke 200 python -c "import __graft_entry__ as g; g.smoke()"
run bench 400 python bench.py --steps 20 --warmup 5
