#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
for C in ${CONFIGS:-c2 c3}; do timeout 300 python scripts/sel_latency.py $C 2>&1 | grep "pdl=1"; done
