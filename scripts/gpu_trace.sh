#!/bin/bash
# per-tile pipeline trace of CTA 0 (debug build) for the configs given
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1 AS_DEBUG_LIB=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
for C in ${CONFIGS:-c4}; do
  for M in ${MODES:-0}; do
    AS_ATTN_DEBUG_MODE=$M timeout 300 python scripts/attn_trace.py --config $C 2>&1 | tail -40
  done
done
