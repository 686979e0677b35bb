"""Build libadaserve.so in-tree with nvcc for sm_100a (no JIT cache, no torch).

    python -m paper_2501_12162_b200.build [--force] [--debug] [-v]

The product library is ``libadaserve.so``.  ``--debug`` (or AS_DEBUG=1) also
builds ``libadaserve_debug.so``: the same sources compiled with -DAS_DEBUG (the
attention/select experiment switches read from the environment, the pipeline
trace) plus the HBM streaming micro-benchmark ``as_debug_stream_bw``
(``include/adaserve_debug.h``).  Nothing on the product path loads it; the
tuning scripts under scripts/ select it with AS_DEBUG_LIB=1.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libadaserve.so")
LIB_DEBUG = os.path.join(PKG, "libadaserve_debug.so")
SOURCES = ["abi.cu", "beam.cu", "sample.cu", "mss.cu", "select.cu", "accept.cu", "attn_simt.cu", "attn_tc.cu", "selftest.cu"]
DEBUG_SOURCES = SOURCES + ["membench.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
PTXAS_LOG = os.path.join(CSRC, "ptxas.log")  # registers / spills of the last build (git-ignored)


def _sources_mtime() -> float:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    deps += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    return max(os.path.getmtime(d) for d in deps)


def _stale(lib: str) -> bool:
    return not os.path.exists(lib) or _sources_mtime() > os.path.getmtime(lib)


def _build_one(lib: str, sources, defines, tag: str):
    def compile_one(src):
        obj = os.path.join(CSRC, f"{src[:-3]}{tag}.o")
        cmd = [NVCC, *FLAGS, *defines, *os.environ.get("AS_NVCC_DEFINES", "").split(), "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, src), "-o",
               obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=min(len(sources), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, sources))
    objs = [o for o, _ in results]
    tmp = lib + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart_static",
           "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return "\n".join(log for _, log in results)


def build(force: bool = False, verbose: bool = False, debug: bool = None) -> str:
    if debug is None:
        debug = os.environ.get("AS_DEBUG") == "1"
    if force or _stale(LIB):
        log = _build_one(LIB, SOURCES, [], "")
        with open(PTXAS_LOG, "w") as f:
            f.write(log)
        if verbose:
            print(log)
    if debug and (force or _stale(LIB_DEBUG)):
        _build_one(LIB_DEBUG, DEBUG_SOURCES, ["-DAS_DEBUG"], ".dbg")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug=("--debug" in sys.argv) or None))
