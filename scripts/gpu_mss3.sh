#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mss" --timeout 120 2>&1 | tail -3
for C in ${CONFIGS:-c2}; do timeout 300 python scripts/mss_run.py --config $C --iters 10 2>&1 | tail -1; done
AS_DEBUG_LIB=1 timeout 300 python scripts/mss_trace.py --config c2 2>&1 | tail -64
