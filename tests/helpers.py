"""Shared helpers for the GPU parity tests (test infrastructure only)."""
import numpy as np
import torch

import oracle
import synth


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def bf16_bits(t):
    """bf16 tensor -> numpy uint16 bit pattern."""
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def workload_to_device(w, dtype):
    keys = ("q", "k_tree", "v_tree", "k_cache", "v_cache")
    out = {k: dev(w[k], dtype) for k in keys}
    out["page_table"] = dev(w["page_table"])
    out["kv_len"] = dev(w["kv_len"])
    out["tree_offsets"] = dev(w["tree_offsets"])
    out["tree_parent"] = dev(w["tree_parent"])
    return out


def oracle_attn(w, scale, requests=None):
    """Oracle attention for all requests, or only for `requests` (a compacted
    sub-problem: their tree rows and only their pages)."""
    if requests is None:
        return oracle.tree_attn(w["q"], w["k_tree"], w["v_tree"], w["k_cache"], w["v_cache"], w["page_table"],
                                w["kv_len"], w["tree_offsets"], w["tree_parent"], scale, n_threads=8)
    to = w["tree_offsets"]
    rows = np.concatenate([np.arange(to[i], to[i + 1]) for i in requests])
    sizes = np.array([to[i + 1] - to[i] for i in requests])
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    pt = w["page_table"][requests]
    used = np.unique(pt[pt >= 0])
    remap = -np.ones(w["k_cache"].shape[0], np.int64)
    remap[used] = np.arange(len(used))
    pt2 = np.where(pt >= 0, remap[np.maximum(pt, 0)], -1).astype(np.int32)
    out, lse = oracle.tree_attn(w["q"][rows], w["k_tree"][rows], w["v_tree"][rows], w["k_cache"][used],
                                w["v_cache"][used], pt2, w["kv_len"][requests], offs, w["tree_parent"][rows], scale,
                                n_threads=8)
    return rows, out, lse
