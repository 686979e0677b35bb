#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/mss_run.py --iters 5 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mss_kernel -s 3 -c 1 \
   -o gpurun_out/prof_mss_${TAG} -f python scripts/mss_run.py --iters 1 > gpurun_out/ncu_mss_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_mss_${TAG}.log
