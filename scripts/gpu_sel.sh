#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "${TESTS:-determin or iteration or select}" --timeout 200 2>&1 | tail -3
for C in ${CONFIGS:-c2 c3}; do AS_DEBUG_LIB=1 timeout 300 python scripts/sel_latency.py $C 2>&1 | grep "pdl=1"; done
