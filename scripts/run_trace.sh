cd "${GRAFT_REPO_ROOT:-/root/repo}"
export AS_DEBUG=1 AS_DEBUG_LIB=1  # debug build (experiment switches)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_tr.log 2>&1 || exit 1
for C in ${CFGS:-c2}; do for W in ${WORLDS:-8}; do
  echo "== $C world $W"
  AS_BENCH_EMULATE_WORLD=$W timeout 200 python scripts/attn_trace.py --config $C 2>&1 | head -12
done; done
