#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m paper_2501_12162_b200.build --debug > /dev/null 2>&1
for C in ${CONFIGS:-c2}; do AS_DEBUG_LIB=1 timeout 300 python scripts/mss_trace.py --config $C 2>&1 | tail -40; done
