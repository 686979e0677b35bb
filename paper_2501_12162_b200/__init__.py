"""B200-native AdaServe hot path: select -> tree-verify attention -> accept.

Thin Python binding over ``libadaserve.so`` (C ABI declared in
``include/adaserve.h``).  This module only marshals torch tensors (device
memory, the current CUDA stream) into the C calls; every step of the path runs
in the library's CUDA kernels.  There is no CPU fallback: if the library is
missing or a tensor is not on a CUDA device, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = ["lib", "select_trees", "select_global_greedy", "select_topm", "select_equal_greedy", "sample_tokens", "mss_verify", "AS_MSS_WALK", "AS_MSS_ALL_NODES", "tree_verify_attn", "AttnSchedule", "parse_schedule", "accept_tokens", "Workspace", "check_device_error",
           "selftest_umma", "AS_ACCEPT_FUSED", "AS_ACCEPT_WALK_ONLY", "AS_ACCEPT_COMMIT_ONLY",
           "AS_ACCEPT_WALK_RECORDS", "AS_ACCEPT_COMMIT_RECORDS", "beam_step", "beam_workspace_size", "AdaServeError",
           "select_workspace_size", "attn_workspace_size", "accept_workspace_size", "DEVICE_ERRORS"]

_PKG = os.path.dirname(os.path.abspath(__file__))
# AS_DEBUG_LIB=1 loads the debug build (experiment switches + tuning instruments,
# include/adaserve_debug.h) -- tuning scripts only; the product path never sets it
LIB_PATH = os.path.join(_PKG, "libadaserve_debug.so" if os.environ.get("AS_DEBUG_LIB") == "1" else "libadaserve.so")

AS_F32, AS_BF16 = 0, 1
AS_ACCEPT_FUSED, AS_ACCEPT_WALK_ONLY, AS_ACCEPT_COMMIT_ONLY = 0, 1, 2
AS_ACCEPT_WALK_RECORDS, AS_ACCEPT_COMMIT_RECORDS = 3, 4
AS_MSS_WALK, AS_MSS_ALL_NODES = 0, 1
DEVICE_ERRORS = {0: "ok", 1: "bad parent", 2: "bad f-hat", 3: "too many candidates", 4: "tree too big",
                 5: "rows overflow", 6: "page overflow", 7: "NaN logit", 8: "path too long", 9: "bad page",
                 10: "bad token", 11: "split-KV pieces not co-resident"}

_c_i32, _c_sz, _vp, _f32 = ctypes.c_int32, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_float
_lib = None


class AdaServeError(RuntimeError):
    pass


def lib():
    """Load libadaserve.so (built in-tree by ``build.py``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise AdaServeError(f"{LIB_PATH} not built: run `python -m paper_2501_12162_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        L.as_status_string.restype = ctypes.c_char_p
        L.as_version.restype = ctypes.c_char_p
        for name in ("as_select_workspace_size", "as_attn_workspace_size", "as_accept_workspace_size",
                     "as_beam_workspace_size"):
            getattr(L, name).restype = _c_sz
        L.as_beam_workspace_size.argtypes = [_c_i32, _c_i32, _c_i32]
        L.as_beam_step.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _vp, _c_i32, _vp, _vp, _vp, _vp, _c_sz, _vp]
        L.as_select_workspace_size.argtypes = [_c_i32, _c_i32]
        L.as_sample_tokens.argtypes = [_c_i32, _c_i32, _vp, _c_i32, _f32, ctypes.c_ulonglong, ctypes.c_ulonglong, _vp,
                                       _vp, _c_sz, _vp]
        L.as_mss_verify.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _c_i32, _vp, _vp, _vp, _c_sz, _vp]
        L.as_attn_workspace_size.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32]
        L.as_accept_workspace_size.argtypes = [_c_i32]
        L.as_select_trees.argtypes = [_c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_i32,
                                      _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_sz, _vp]
        L.as_select_topm.argtypes = [_c_i32, _c_i32, _vp, _vp, _vp, _vp, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _c_sz, _vp]
        L.as_tree_verify_attn.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp,
                                          _c_i32, _c_i32, _vp, _c_i32, _vp, _vp, _vp, _f32, _vp, _vp, _vp, _c_sz,
                                          _vp]
        L.as_tree_verify_attn_sched.argtypes = L.as_tree_verify_attn.argtypes + [_vp]
        L.as_accept_tokens.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _c_i32,
                                       _c_i32, _c_i32, _vp, _vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_i32, _vp, _vp,
                                       _c_i32, _c_i32, _vp, _c_i32, _vp, _vp, _vp, _c_sz, _vp]
        L.as_check_device_error.argtypes = [_vp, _vp, _vp, _vp]
        L.as_reset_workspace.argtypes = [_vp, _c_sz, _vp]
        L.as_selftest_umma.argtypes = [_vp, _vp, _vp, _c_i32, _c_i32, _c_i32, _vp]
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise AdaServeError(f"{what}: {lib().as_status_string(status).decode()} (status {status})")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise AdaServeError("tensors must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise AdaServeError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dt(t):
    if t.dtype == torch.bfloat16:
        return AS_BF16
    if t.dtype == torch.float32:
        return AS_F32
    raise AdaServeError(f"unsupported dtype {t.dtype}")


def _need(t, dtype, name):
    if t.dtype != dtype:
        raise AdaServeError(f"{name} must be {dtype}, got {t.dtype}")


def beam_workspace_size(n_req, width, vocab):
    return int(lib().as_beam_workspace_size(n_req, width, vocab))


def beam_step(layer, width, draft_probs, cand_parent, cand_prob, cand_token, cand_stride, workspace=None):
    """as_beam_step: speculation layer `layer` (Step 1) for every
    request, written in place into the candidate forest (stride cand_stride).
    draft_probs [n_req, w_in, vocab] fp32, w_in = 1 at layer 1 else width."""
    _need(draft_probs, torch.float32, "draft_probs")
    n, w_in, vocab = draft_probs.shape
    if w_in != (1 if layer == 1 else width):
        raise AdaServeError(f"draft_probs must have {1 if layer == 1 else width} rows per request at layer {layer}")
    _need(cand_parent, torch.int32, "cand_parent")
    _need(cand_prob, torch.float32, "cand_prob")
    _need(cand_token, torch.int32, "cand_token")
    ws = workspace if workspace is not None else Workspace(beam_workspace_size(n, width, vocab), draft_probs.device)
    ws.ensure(beam_workspace_size(n, width, vocab))
    _check(lib().as_beam_step(n, layer, width, vocab, _ptr(draft_probs), cand_stride, _ptr(cand_parent),
                              _ptr(cand_prob), _ptr(cand_token), ws.ptr, ws.nbytes, _stream()), "as_beam_step")
    return ws


def sample_tokens(logits, inv_temperature, seed, offset=0, out=None, workspace=None):
    """as_sample_tokens (NEXT-3(a), reading R23): one Gumbel-max sample of
    softmax(logits * inv_temperature) per row of logits [rows, vocab] (fp32 or
    bf16, device); returns int32 [rows] -- the per-node target samples of the
    stochastic walk (pass them as accept_tokens' target_tokens)."""
    if logits.dtype not in (torch.float32, torch.bfloat16) or logits.dim() != 2 or not logits.is_contiguous():
        raise AdaServeError("logits must be a contiguous [rows, vocab] fp32/bf16 tensor")
    rows, vocab = logits.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.int32, device=logits.device)
    ws = workspace if workspace is not None else Workspace(256, logits.device)
    _check(lib().as_sample_tokens(rows, vocab, _ptr(logits), 1 if logits.dtype == torch.bfloat16 else 0,
                                  float(inv_temperature), int(seed) & (2**64 - 1), int(offset) & (2**64 - 1),
                                  _ptr(out), ws.ptr, ws.nbytes, _stream()), "as_sample_tokens")
    return out, ws


def mss_verify(tree_offsets, tree_parent, tree_tokens, target_probs, draft_probs, uniforms, bonus_uniforms,
               max_path=None, mode=AS_MSS_WALK, req_range=None, records=None, emitted=None, workspace=None):
    """as_mss_verify (NEXT-3(b), reading R25): SpecInfer multi-step speculative
    sampling over trees of drawn drafts.  target_probs / draft_probs: fp32
    [rows, vocab]; uniforms / bonus_uniforms: fp32 [rows] in (0, 1].
    mode AS_MSS_WALK: returns (records int32 [n, max_path + 2] = {len, bonus,
    path}, emitted int32 [rows] (-1 off the path), workspace); commit with
    accept_tokens(AS_ACCEPT_COMMIT_RECORDS).  mode AS_MSS_ALL_NODES: records is
    None and emitted holds every node's token."""
    for t in (target_probs, draft_probs):
        if t.dtype != torch.float32 or t.dim() != 2 or not t.is_contiguous():
            raise AdaServeError("target_probs / draft_probs must be contiguous fp32 [rows, vocab]")
    if uniforms.dtype != torch.float32 or bonus_uniforms.dtype != torch.float32:
        raise AdaServeError("uniforms must be fp32")
    n = tree_offsets.numel() - 1
    rows, vocab = target_probs.shape
    b, e = (0, n) if req_range is None else req_range
    dev = target_probs.device
    if max_path is None:
        max_path = 256
    if mode == AS_MSS_WALK and records is None:
        records = torch.empty((n, max_path + 2), dtype=torch.int32, device=dev)
    if emitted is None:
        emitted = torch.empty(rows, dtype=torch.int32, device=dev)
    ws = workspace if workspace is not None else Workspace(256, dev)
    _check(lib().as_mss_verify(mode, n, b, e, rows, vocab, _ptr(tree_offsets), _ptr(tree_parent), _ptr(tree_tokens),
                               _ptr(target_probs), _ptr(draft_probs), _ptr(uniforms), _ptr(bonus_uniforms),
                               max_path, _ptr(records) if records is not None else None, _ptr(emitted), ws.ptr,
                               ws.nbytes, _stream()), "as_mss_verify")
    return (records if mode == AS_MSS_WALK else None), emitted, ws


def select_workspace_size(n_req, n_cand_total):
    return int(lib().as_select_workspace_size(n_req, n_cand_total))


def attn_workspace_size(dtype, n_req, n_tree_rows, n_q, head_dim, max_kv_len):
    return int(lib().as_attn_workspace_size(dtype, n_req, n_tree_rows, n_q, head_dim, max_kv_len))


def accept_workspace_size(n_tree_rows):
    return int(lib().as_accept_workspace_size(n_tree_rows))


class Workspace:
    """A zero-initialised device scratch buffer (the C ABI's `workspace`)."""

    def __init__(self, nbytes: int, device=None):
        self.nbytes = max(256, int(nbytes))
        self.buf = torch.zeros(self.nbytes + 256, dtype=torch.uint8, device=device or "cuda")
        off = (-self.buf.data_ptr()) % 256
        self.view = self.buf[off:off + self.nbytes]

    @property
    def ptr(self):
        return ctypes.c_void_p(self.view.data_ptr())

    def ensure(self, nbytes):
        if nbytes > self.nbytes:
            self.__init__(nbytes, self.buf.device)
        return self


def check_device_error(ws: Workspace):
    code, req = ctypes.c_int32(0), ctypes.c_int32(0)
    _check(lib().as_check_device_error(ws.ptr, ctypes.byref(code), ctypes.byref(req), _stream()), "check")
    return code.value, req.value


# ---------------------------------------------------------------------------
def select_trees(cand_offsets, cand_parent, cand_prob, slo_deficit, depth_d, n_max, budget, cand_token=None,
                 n_cand_total=None, out=None, workspace=None):
    """as_select_trees (Alg. 2).  Inputs are device tensors:
    cand_offsets/cand_parent int32, cand_prob float32, slo_deficit float64,
    cand_token int32 or None.  Returns dict of device int32 tensors
    (tree_offsets [n+1], tree_parent/tree_src/tree_depth/tree_token [budget],
    slo_count [n]).  `n_cand_total` is the host-known size of cand_prob."""
    n = cand_offsets.numel() - 1
    _need(cand_offsets, torch.int32, "cand_offsets")
    _need(cand_parent, torch.int32, "cand_parent")
    _need(cand_prob, torch.float32, "cand_prob")
    _need(slo_deficit, torch.float64, "slo_deficit")
    N = cand_prob.numel() if n_cand_total is None else int(n_cand_total)
    dev = cand_prob.device
    if out is None:
        cap = max(int(budget), 1)
        out = dict(tree_offsets=torch.empty(n + 1, dtype=torch.int32, device=dev),
                   tree_parent=torch.empty(cap, dtype=torch.int32, device=dev),
                   tree_src=torch.empty(cap, dtype=torch.int32, device=dev),
                   tree_depth=torch.empty(cap, dtype=torch.int32, device=dev),
                   tree_token=torch.empty(cap, dtype=torch.int32, device=dev) if cand_token is not None else None,
                   slo_count=torch.empty(max(n, 1), dtype=torch.int32, device=dev))
    ws = workspace if workspace is not None else Workspace(select_workspace_size(n, N), dev)
    ws.ensure(select_workspace_size(n, N))
    st = lib().as_select_trees(n, N, _ptr(cand_offsets), _ptr(cand_parent), _ptr(cand_prob), _ptr(cand_token),
                               _ptr(slo_deficit), depth_d, n_max, int(budget), _ptr(out["tree_offsets"]),
                               _ptr(out["tree_parent"]), _ptr(out["tree_src"]), _ptr(out.get("tree_depth")),
                               _ptr(out.get("tree_token")), _ptr(out.get("slo_count")), ws.ptr, ws.nbytes,
                               _stream())
    _check(st, "as_select_trees")
    out["workspace"] = ws
    return out



def select_global_greedy(cand_offsets, cand_parent, cand_prob, budget, cand_token=None, out=None, workspace=None):
    """GlobalGreedy (the paper's ablation) as a
    parameterisation of as_select_trees: with every A(r) <= 1 the SLO stage
    takes nothing (1 + sum f-hat < A_cap never holds), so after the roots the
    whole budget goes to the global top-(B - n) candidates by (f-hat desc,
    request asc, index asc).  Same kernel, same launch."""
    n = cand_offsets.numel() - 1
    zeros = torch.zeros(max(n, 1), dtype=torch.float64, device=cand_prob.device)[:n]
    return select_trees(cand_offsets, cand_parent, cand_prob, zeros, 0, 0, budget, cand_token=cand_token, out=out,
                        workspace=workspace)

def select_topm(cand_offsets, cand_parent, cand_prob, m_base, m_extra=0, cand_token=None, out=None,
                workspace=None):
    """as_select_topm (NEXT-4, reading R24): request i keeps its root and its
    best min(m_base + (i < m_extra), C_i - 1) candidates by (f-hat desc, index
    asc).  Eagle-2 top-m: select_topm(..., m); EqualGreedy: select_equal_greedy.
    Returns the same dict as select_trees ('kept' instead of 'slo_count')."""
    n = cand_offsets.numel() - 1
    _need(cand_offsets, torch.int32, "cand_offsets")
    _need(cand_parent, torch.int32, "cand_parent")
    _need(cand_prob, torch.float32, "cand_prob")
    N = cand_prob.numel()
    dev = cand_prob.device
    if out is None:
        cap = max(1, n + n * int(m_base) + int(m_extra))
        cap = min(cap, max(N, 1))
        out = dict(tree_offsets=torch.empty(n + 1, dtype=torch.int32, device=dev),
                   tree_parent=torch.empty(cap, dtype=torch.int32, device=dev),
                   tree_src=torch.empty(cap, dtype=torch.int32, device=dev),
                   tree_depth=torch.empty(cap, dtype=torch.int32, device=dev),
                   tree_token=torch.empty(cap, dtype=torch.int32, device=dev) if cand_token is not None else None,
                   kept=torch.empty(max(n, 1), dtype=torch.int32, device=dev))
    ws = workspace if workspace is not None else Workspace(select_workspace_size(n, N), dev)
    ws.ensure(select_workspace_size(n, N))
    st = lib().as_select_topm(n, N, _ptr(cand_offsets), _ptr(cand_parent), _ptr(cand_prob), _ptr(cand_token),
                              int(m_base), int(m_extra), _ptr(out["tree_offsets"]), _ptr(out["tree_parent"]),
                              _ptr(out["tree_src"]), _ptr(out.get("tree_depth")), _ptr(out.get("tree_token")),
                              _ptr(out.get("kept")), ws.ptr, ws.nbytes, _stream())
    _check(st, "as_select_topm")
    out["workspace"] = ws
    return out


def select_equal_greedy(cand_offsets, cand_parent, cand_prob, budget, cand_token=None, out=None, workspace=None):
    """EqualGreedy (reading R24): the budget B (roots included, R1)
    split evenly -- floor(B/n) nodes per request, one more for the first B mod n
    requests -- each request filling its share greedily by f-hat."""
    n = cand_offsets.numel() - 1
    if budget < n:
        raise AdaServeError("budget smaller than the number of requests (R10)")
    if n == 0:
        return select_topm(cand_offsets, cand_parent, cand_prob, 0, 0, cand_token, out, workspace)
    return select_topm(cand_offsets, cand_parent, cand_prob, budget // n - 1, budget % n, cand_token, out, workspace)


class AttnSchedule(ctypes.Structure):
    """as_attn_schedule: q_tiles_per_cta (0 auto, 1, 2), cluster_ctas (0/1, 2, 4),
    split (-1 auto, 0 whole units only, 1 allowed), cta_pair (1: cta_group::2 pairs)
    -- A/B overrides, results identical."""
    _fields_ = [("q_tiles_per_cta", ctypes.c_int32), ("cluster_ctas", ctypes.c_int32), ("split", ctypes.c_int32),
                ("cta_pair", ctypes.c_int32)]


def parse_schedule(spec):
    """'nq=2,cs=1,split=0' (any subset) -> AttnSchedule; None/'' -> None."""
    if not spec:
        return None
    s = AttnSchedule(0, 0, -1, 0)
    for kv in str(spec).split(","):
        k, v = kv.split("=")
        setattr(s, {"nq": "q_tiles_per_cta", "cs": "cluster_ctas", "split": "split", "pair": "cta_pair"}[k.strip()],
                int(v))
    return s


def tree_verify_attn(q, k_tree, v_tree, k_cache, v_cache, page_table, kv_len, tree_offsets, tree_parent, sm_scale,
                     want_lse=False, out=None, lse=None, workspace=None, schedule=None):
    """as_tree_verify_attn.  q [R, n_q, d], k_tree/v_tree [R, n_kv, d],
    caches [pages, n_kv, page_size, d] (bf16 -> tcgen05 path, fp32 -> SIMT path),
    page_table [n, max_pages] int32, kv_len [n] int32.  Returns (out, lse).
    schedule: None, an AttnSchedule, or a parse_schedule string (A/B only)."""
    if isinstance(schedule, str):
        schedule = parse_schedule(schedule)
    R, n_q, d = q.shape
    n_kv = k_tree.shape[1]
    n = tree_offsets.numel() - 1
    dt = _dt(q)
    for t, name in ((k_tree, "k_tree"), (v_tree, "v_tree"), (k_cache, "k_cache"), (v_cache, "v_cache")):
        _need(t, q.dtype, name)
    _need(page_table, torch.int32, "page_table")
    _need(kv_len, torch.int32, "kv_len")
    if out is None:
        out = torch.empty_like(q)
    if want_lse and lse is None:
        lse = torch.empty((R, n_q), dtype=torch.float32, device=q.device)
    ws = workspace if workspace is not None else Workspace(attn_workspace_size(dt, n, R, n_q, d, 0), q.device)
    st = lib().as_tree_verify_attn_sched(dt, n, R, n_q, n_kv, d, _ptr(q), _ptr(k_tree), _ptr(v_tree),
                                         _ptr(k_cache), _ptr(v_cache), k_cache.shape[0], k_cache.shape[2],
                                         _ptr(page_table), page_table.shape[1] if page_table.dim() == 2 else 0,
                                         _ptr(kv_len), _ptr(tree_offsets), _ptr(tree_parent), float(sm_scale),
                                         _ptr(out), _ptr(lse if want_lse else None), ws.ptr, ws.nbytes, _stream(),
                                         ctypes.byref(schedule) if schedule is not None else None)
    _check(st, "as_tree_verify_attn")
    return out, (lse if want_lse else None)


def accept_tokens(phase, tree_offsets, tree_parent=None, tree_tokens=None, target_tokens=None, target_logits=None,
                  max_path=16, k_tree=None, v_tree=None, k_cache=None, v_cache=None, page_table=None, kv_len=None,
                  req_range=None, accept_len=None, accept_path=None, bonus_token=None, n_tree_rows=None,
                  workspace=None, kv_len_out=None):
    """as_accept_tokens (walk + commit).  Returns dict(accept_len,
    accept_path, bonus_token); for FUSED / COMMIT_ONLY the caches are updated
    in place and the new lengths go to kv_len_out (None: kv_len in place)."""
    n = tree_offsets.numel() - 1
    dev = tree_offsets.device
    b, e = (0, n) if req_range is None else req_range
    R = int(n_tree_rows if n_tree_rows is not None else
            (tree_parent.numel() if tree_parent is not None else (k_tree.shape[0] if k_tree is not None else 0)))
    records = phase in (AS_ACCEPT_WALK_RECORDS, AS_ACCEPT_COMMIT_RECORDS)
    if records:
        # accept_path = int32 [rows >= n, 2 + max_path] records {len, bonus, path}
        if accept_path is None:
            accept_path = torch.empty((max(n, 1), 2 + max_path), dtype=torch.int32, device=dev)
        if accept_path.dim() != 2 or accept_path.shape[0] < n or accept_path.shape[1] != 2 + max_path:
            raise AdaServeError("records must be int32 [>= n_req, 2 + max_path]")
    else:
        if accept_len is None:
            accept_len = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        if accept_path is None:
            accept_path = torch.empty((max(n, 1), max_path), dtype=torch.int32, device=dev)
        if bonus_token is None:
            bonus_token = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ws = workspace if workspace is not None else Workspace(accept_workspace_size(R), dev)
    ws.ensure(accept_workspace_size(R))
    kv_dt = _dt(k_tree) if k_tree is not None else AS_BF16
    lg_dt = _dt(target_logits) if target_logits is not None else AS_F32
    vocab = target_logits.shape[1] if target_logits is not None else 0
    n_kv = k_tree.shape[1] if k_tree is not None else 0
    d = k_tree.shape[2] if k_tree is not None else 0
    st = lib().as_accept_tokens(phase, n, b, e, R, _ptr(tree_offsets), _ptr(tree_parent), _ptr(tree_tokens),
                                _ptr(target_tokens), _ptr(target_logits), lg_dt, vocab, max_path, _ptr(accept_len),
                                _ptr(accept_path), _ptr(bonus_token), _ptr(k_tree), _ptr(v_tree), kv_dt, n_kv, d,
                                _ptr(k_cache), _ptr(v_cache), k_cache.shape[0] if k_cache is not None else 0,
                                k_cache.shape[2] if k_cache is not None else 0, _ptr(page_table),
                                page_table.shape[1] if page_table is not None else 0, _ptr(kv_len), _ptr(kv_len_out),
                                ws.ptr, ws.nbytes,
                                _stream())
    _check(st, "as_accept_tokens")
    if records:
        return dict(records=accept_path, workspace=ws)
    return dict(accept_len=accept_len, accept_path=accept_path, bonus_token=bonus_token, workspace=ws)


def selftest_umma(a, b, n, k, b_mn_major):
    """Debug: D = A . B^T (or A . B for MN-major B) through tcgen05 (see adaserve.h)."""
    d = torch.empty((256 if b_mn_major & 4 else 128, n), dtype=torch.float32, device=a.device)
    _check(lib().as_selftest_umma(_ptr(a), _ptr(b), _ptr(d), n, k, int(b_mn_major), _stream()), "selftest")
    return d
