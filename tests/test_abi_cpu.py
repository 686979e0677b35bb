"""The C-ABI library loads on a CPU-only box, exports every symbol the header
declares, and rejects host-checkable bad arguments without launching."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "adaserve.h")


@pytest.fixture(scope="module")
def L():
    from paper_2501_12162_b200 import build as b
    b.build()
    import paper_2501_12162_b200 as pk
    return pk.lib()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(as_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert "as_select_trees" in names and "as_tree_verify_attn" in names and "as_accept_tokens" in names
    for n in names:
        assert hasattr(L, n), n
    nm = os.popen(f"nm -D {os.path.join(ROOT, 'paper_2501_12162_b200', 'libadaserve.so')}").read()
    for n in names:
        assert re.search(rf"\bT {n}\b", nm), n


def test_status_strings_and_sizes(L):
    assert L.as_status_string(0).decode() == "ok"
    assert "budget" in L.as_status_string(2).decode()
    assert L.as_version().decode().startswith("adaserve-b200")
    assert L.as_select_workspace_size(256, 16640) >= 16640 * 8
    assert L.as_accept_workspace_size(4096) >= 4096 * 4
    assert L.as_attn_workspace_size(1, 64, 2048, 32, 128, 2048) >= 256


def test_host_checks_return_without_launch(L):
    vp = ctypes.c_void_p
    dummy = vp(4096)
    # budget < n_req -> AS_ERR_BUDGET_TOO_SMALL (R10)
    st = L.as_select_trees(4, 8, dummy, dummy, dummy, None, dummy, 3, 3, 3, dummy, dummy, dummy, None, None, None,
                           dummy, 1 << 20, None)
    assert st == 2
    # as_select_topm: m_extra outside [0, n_req] / negative m_base -> AS_ERR_INVALID_ARG
    f = L.as_select_topm
    f.argtypes = [ctypes.c_int32, ctypes.c_int32] + [vp] * 4 + [ctypes.c_int32] * 2 + [vp] * 7 + [ctypes.c_size_t, vp]
    assert f(4, 8, dummy, dummy, dummy, None, 1, 5, dummy, dummy, dummy, None, None, None, dummy, 1 << 20, None) == 1
    assert f(4, 8, dummy, dummy, dummy, None, -1, 0, dummy, dummy, dummy, None, None, None, dummy, 1 << 20, None) == 1
    assert f(4, 8, dummy, dummy, dummy, None, 1, 0, dummy, dummy, dummy, None, None, None, None, 0, None) == 4
    # unsupported head_dim -> AS_ERR_UNSUPPORTED
    st = L.as_tree_verify_attn(1, 1, 8, 4, 4, 96, dummy, dummy, dummy, dummy, dummy, 4, 16, dummy, 4, dummy,
                               dummy, dummy, ctypes.c_float(0.1), dummy, None, vp(256 * 64), 256, None)
    assert st == 3
    # n_q % n_kv != 0
    st = L.as_tree_verify_attn(1, 1, 8, 6, 4, 128, dummy, dummy, dummy, dummy, dummy, 4, 16, dummy, 4, dummy,
                               dummy, dummy, ctypes.c_float(0.1), dummy, None, vp(256 * 64), 256, None)
    assert st == 3
    # misaligned workspace
    st = L.as_tree_verify_attn(1, 1, 8, 4, 4, 128, dummy, dummy, dummy, dummy, dummy, 4, 16, dummy, 4, dummy,
                               dummy, dummy, ctypes.c_float(0.1), dummy, None, vp(256 * 64 + 4), 256, None)
    assert st == 4
    # accept: bad phase / max_path
    st = L.as_accept_tokens(7, 1, 0, 1, 4, dummy, dummy, dummy, dummy, None, 0, 0, 8, dummy, dummy, dummy,
                            None, None, 1, 0, 0, None, None, 0, 0, None, 0, None, None, vp(1 << 16), 1 << 12, None)
    assert st == 1
    st = L.as_accept_tokens(1, 1, 0, 1, 4, dummy, dummy, dummy, dummy, None, 0, 0, 65, dummy, dummy, dummy,
                            None, None, 1, 0, 0, None, None, 0, 0, None, 0, None, None, vp(1 << 16), 1 << 12, None)
    assert st == 3


def test_product_path_does_not_import_oracle():
    """The product package never imports / links anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2501_12162_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f
                assert "adaserve_ref" not in src, f


def test_sample_tokens_host_checks(L):
    """as_sample_tokens rejects bad host arguments before any launch."""
    f = L.as_sample_tokens
    f.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_float,
                  ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                  ctypes.c_void_p]
    assert f(0, 10, None, 0, 1.0, 1, 0, None, None, 0, None) == 0          # nothing to do
    assert f(-1, 10, None, 0, 1.0, 1, 0, None, None, 0, None) != 0         # negative rows
    assert f(2, 10, None, 0, 1.0, 1, 0, None, None, 0, None) != 0          # null logits
    assert f(2, 10, 256, 0, -1.0, 1, 0, 512, 768, 256, None) != 0          # negative inv_temperature
    assert f(2, 10, 256, 5, 1.0, 1, 0, 512, 768, 256, None) != 0           # unknown dtype


def test_mss_verify_host_checks(L):
    """as_mss_verify rejects bad host arguments before any launch."""
    f = L.as_mss_verify
    vp, i32 = ctypes.c_void_p, ctypes.c_int32
    f.argtypes = [i32] * 6 + [vp] * 7 + [i32, vp, vp, vp, ctypes.c_size_t, vp]
    d = 4096
    args = lambda mode=0, n=2, b=0, e=2, vocab=1000, mp=8, rec=d, em=d, ws=1 << 16: (
        mode, n, b, e, 16, vocab, d, d, d, d, d, d, d, mp, rec, em, ws, 256, None)
    assert f(*args(mode=2)) == 1                 # unknown mode
    assert f(*args(e=3)) == 1                    # req_end > n_req
    assert f(*args(b=2, e=2)) == 0               # empty range: nothing to do
    assert f(*args(vocab=400000)) == 3           # vocab beyond two 16-CTA clusters' shared memory
    assert f(*args(mp=0)) == 1                   # walk needs max_path >= 1
    assert f(*args(rec=None, em=None)) == 1      # walk needs an output
    assert f(*args(mode=1, em=None)) == 1        # all-nodes needs emitted
    assert f(*args(ws=(1 << 16) + 4)) == 4       # misaligned workspace
