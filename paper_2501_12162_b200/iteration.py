"""NEXT-2: the whole verify iteration as one replayed CUDA graph,
keyed by its shapes, plus the paper's adaptive (d, w) host policy.

* ``adaptive_params`` -- P:L880-884 ("Adaptive control"):
      d = clip(D_max, D_min, floor(B_1 / (n + c_1)) - 1)
      w = clip(W_max, 1,     floor(B_2 / n) + c_2)
  with clip(hi, lo, x) = max(lo, min(hi, x)).
* ``IterationGraph`` -- select -> tree-verify attention -> accept (+ commit)
  captured once per shape key (n, d, w, budget, rows, heads, ...) and replayed
  (CUDA graphs need identical shapes; across iterations with the
  same n, d, w the shapes repeat).  The graph holds static input/output
  tensors; a caller copies the iteration's inputs in (or writes them in place)
  and replays.  Every kernel is the library's (``select_trees``,
  ``tree_verify_attn``, ``accept_tokens``); the graph only removes the host
  launch path.  The three kernels are launched with programmatic dependent
  launch, which a captured graph keeps.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch


def adaptive_params(n_active: int, d_max: int, d_min: int, w_max: int, b1: int, b2: int, c1: int = 0,
                    c2: int = 0):
    """(d, w) for the next iteration from the number of active requests."""
    if n_active < 1:
        raise ValueError("n_active must be >= 1")

    def clip(hi, lo, x):
        return max(lo, min(hi, x))
    d = clip(d_max, d_min, b1 // (n_active + c1) - 1)
    w = clip(w_max, 1, b2 // n_active + c2)
    return d, w


@dataclass
class IterationShape:
    """Everything that fixes the kernels' launch shapes (the graph cache key)."""
    n_req: int
    n_cand: int          # candidates in the forest (1 + d*w per request for a beam forest)
    depth_d: int
    n_max: int
    budget: int          # tree rows (sum K_i <= budget)
    n_q: int
    n_kv: int
    head_dim: int
    num_pages: int
    page_size: int
    max_pages: int
    max_path: int
    dtype: torch.dtype = torch.bfloat16

    def key(self):
        return (self.n_req, self.n_cand, self.depth_d, self.n_max, self.budget, self.n_q, self.n_kv, self.head_dim,
                self.num_pages, self.page_size, self.max_pages, self.max_path, self.dtype)


@dataclass
class IterationGraph:
    """Static buffers + a captured CUDA graph of one verify iteration."""
    shape: IterationShape
    sm_scale: float
    device: torch.device = field(default_factory=lambda: torch.device("cuda"))

    def __post_init__(self):
        import paper_2501_12162_b200 as ada
        s, dev = self.shape, self.device
        i32 = dict(dtype=torch.int32, device=dev)
        self.inputs = dict(
            cand_offsets=torch.zeros(s.n_req + 1, **i32), cand_parent=torch.zeros(s.n_cand, **i32),
            cand_prob=torch.ones(s.n_cand, dtype=torch.float32, device=dev), cand_token=torch.zeros(s.n_cand, **i32),
            slo_deficit=torch.zeros(s.n_req, dtype=torch.float64, device=dev),
            q=torch.zeros((s.budget, s.n_q, s.head_dim), dtype=s.dtype, device=dev),
            k_tree=torch.zeros((s.budget, s.n_kv, s.head_dim), dtype=s.dtype, device=dev),
            v_tree=torch.zeros((s.budget, s.n_kv, s.head_dim), dtype=s.dtype, device=dev),
            target_tokens=torch.zeros(s.budget, **i32),
            k_cache=torch.zeros((s.num_pages, s.n_kv, s.page_size, s.head_dim), dtype=s.dtype, device=dev),
            v_cache=torch.zeros((s.num_pages, s.n_kv, s.page_size, s.head_dim), dtype=s.dtype, device=dev),
            page_table=torch.full((s.n_req, s.max_pages), -1, **i32), kv_len=torch.zeros(s.n_req, **i32))
        self.outputs = dict(
            tree_offsets=torch.zeros(s.n_req + 1, **i32), tree_parent=torch.zeros(s.budget, **i32),
            tree_src=torch.zeros(s.budget, **i32), tree_depth=torch.zeros(s.budget, **i32),
            tree_token=torch.zeros(s.budget, **i32), slo_count=torch.zeros(s.n_req, **i32),
            out=torch.zeros((s.budget, s.n_q, s.head_dim), dtype=s.dtype, device=dev),
            accept_len=torch.zeros(s.n_req, **i32), accept_path=torch.zeros((s.n_req, s.max_path), **i32),
            bonus_token=torch.zeros(s.n_req, **i32), kv_len_out=torch.zeros(s.n_req, **i32))
        self.ws = dict(select=ada.Workspace(ada.select_workspace_size(s.n_req, s.n_cand), dev),
                       attn=ada.Workspace(ada.attn_workspace_size(0 if s.dtype == torch.float32 else 1, s.n_req,
                                                                  s.budget, s.n_q, s.head_dim, 0), dev),
                       accept=ada.Workspace(ada.accept_workspace_size(s.budget), dev))
        self.graph = None

    def _run(self):
        import paper_2501_12162_b200 as ada
        I, O, s = self.inputs, self.outputs, self.shape
        sel = dict(tree_offsets=O["tree_offsets"], tree_parent=O["tree_parent"], tree_src=O["tree_src"],
                   tree_depth=O["tree_depth"], tree_token=O["tree_token"], slo_count=O["slo_count"])
        ada.select_trees(I["cand_offsets"], I["cand_parent"], I["cand_prob"], I["slo_deficit"], s.depth_d, s.n_max,
                         s.budget, cand_token=I["cand_token"], out=sel, workspace=self.ws["select"])
        ada.tree_verify_attn(I["q"], I["k_tree"], I["v_tree"], I["k_cache"], I["v_cache"], I["page_table"],
                             I["kv_len"], O["tree_offsets"], O["tree_parent"], self.sm_scale, out=O["out"],
                             workspace=self.ws["attn"])
        ada.accept_tokens(ada.AS_ACCEPT_FUSED, O["tree_offsets"], O["tree_parent"], O["tree_token"],
                          target_tokens=I["target_tokens"], max_path=s.max_path, k_tree=I["k_tree"],
                          v_tree=I["v_tree"], k_cache=I["k_cache"], v_cache=I["v_cache"],
                          page_table=I["page_table"], kv_len=I["kv_len"], kv_len_out=O["kv_len_out"],
                          accept_len=O["accept_len"], accept_path=O["accept_path"], bonus_token=O["bonus_token"],
                          n_tree_rows=s.budget, workspace=self.ws["accept"])

    def _reset_workspaces(self):
        # the warm-up runs on whatever the static inputs hold (zeros before the
        # caller fills them) and may leave sticky device-error words: clear them
        # so as_check_device_error reports only what real iterations cause
        for ws in self.ws.values():
            ws.view.zero_()

    def capture(self):
        """Warm up eagerly (first-use attribute setup), then capture."""
        self._run()
        torch.cuda.synchronize()
        self._reset_workspaces()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._run()
        torch.cuda.synchronize()
        self._reset_workspaces()
        return self

    def replay(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()
        return self.outputs


class GraphCache:
    """IterationGraph per shape key (n, d, w, budget, ...): built on first use."""

    def __init__(self, sm_scale: float, device=None):
        self.sm_scale = sm_scale
        self.device = device or torch.device("cuda")
        self.graphs = {}

    def get(self, shape: IterationShape) -> IterationGraph:
        k = shape.key()
        if k not in self.graphs:
            self.graphs[k] = IterationGraph(shape, self.sm_scale, self.device).capture()
        return self.graphs[k]
