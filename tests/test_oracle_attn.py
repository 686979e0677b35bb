"""Pins for the explicit-mask tree-attention oracle (O4).

The oracle is checked against independent formulations: torch CPU SDPA with
is_causal for chain trees (P-att-1), a numpy decode-attention for root-only
trees (P-att-2), and closed forms (P-att-3/4); structural properties (page
permutation, GQA head mapping, sibling permutation) are checked bit-exactly.
"""
import numpy as np
import pytest
import torch

import oracle
import synth


def _wl(rng, sizes, kv_lens, n_q=4, n_kv=4, d=64, page_size=16, shape="random", bf16=False):
    return synth.tree_workload(rng, sizes, kv_lens, n_q, n_kv, d, page_size, shape=shape, bf16=bf16)


def _run(w, scale=None):
    d = w["q"].shape[2]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    return oracle.tree_attn(w["q"], w["k_tree"], w["v_tree"], w["k_cache"], w["v_cache"], w["page_table"],
                            w["kv_len"], w["tree_offsets"], w["tree_parent"], np.float32(scale))


def _dense_prefix(w, i, kvh):
    L = int(w["kv_len"][i])
    ps = w["k_cache"].shape[2]
    ks = [w["k_cache"][w["page_table"][i, t // ps], kvh, t % ps] for t in range(L)]
    vs = [w["v_cache"][w["page_table"][i, t // ps], kvh, t % ps] for t in range(L)]
    d = w["k_cache"].shape[3]
    return (np.array(ks, np.float64).reshape(L, d), np.array(vs, np.float64).reshape(L, d))


@pytest.mark.parametrize("G", [1, 2])
def test_chain_equals_causal_sdpa(G):
    """P-att-1: a chain tree is ordinary causal decoding of L+K tokens."""
    rng = np.random.default_rng(1)
    n_kv = 2
    w = _wl(rng, [6, 1, 9], [37, 0, 64], n_q=n_kv * G, n_kv=n_kv, d=32, page_size=16, shape="chain")
    out, lse = _run(w)
    to = w["tree_offsets"]
    for i in range(3):
        K = to[i + 1] - to[i]
        L = int(w["kv_len"][i])
        for h in range(n_kv * G):
            kvh = h // G
            kp, vp = _dense_prefix(w, i, kvh)
            k = np.concatenate([kp, w["k_tree"][to[i]:to[i + 1], kvh].astype(np.float64)])
            v = np.concatenate([vp, w["v_tree"][to[i]:to[i + 1], kvh].astype(np.float64)])
            q = np.zeros((L + K, k.shape[1]))
            q[L:] = w["q"][to[i]:to[i + 1], h]
            ref = torch.nn.functional.scaled_dot_product_attention(
                torch.from_numpy(q)[None, None], torch.from_numpy(k)[None, None],
                torch.from_numpy(v)[None, None], is_causal=True)[0, 0, L:].numpy()
            np.testing.assert_allclose(out[to[i]:to[i + 1], h], ref, rtol=0, atol=2e-6)


def test_root_only_is_decode_attention():
    """P-att-2: a root-only tree is single-token decode over L+1 keys (numpy softmax)."""
    rng = np.random.default_rng(2)
    w = _wl(rng, [1, 1], [50, 129], n_q=4, n_kv=2, d=64, page_size=32)
    out, lse = _run(w)
    for i in range(2):
        for h in range(4):
            kp, vp = _dense_prefix(w, i, h // 2)
            k = np.vstack([kp, w["k_tree"][i, h // 2][None].astype(np.float64)])
            v = np.vstack([vp, w["v_tree"][i, h // 2][None].astype(np.float64)])
            s = k @ w["q"][i, h].astype(np.float64) / np.sqrt(64)
            p = np.exp(s - s.max())
            np.testing.assert_allclose(out[i, h], p @ v / p.sum(), atol=2e-6, rtol=0)
            np.testing.assert_allclose(lse[i, h], np.log(np.exp(s).sum()), rtol=1e-6)


def test_closed_forms():
    """P-att-3: L=0, one node -> O = v_root exactly.  P-att-4: constant V -> O = c;
    equal K rows -> uniform weights -> mean of the allowed V rows."""
    rng = np.random.default_rng(3)
    w = _wl(rng, [1], [0], n_q=2, n_kv=1, d=16, page_size=16)
    out, _ = _run(w)
    np.testing.assert_array_equal(out[0, 0], w["v_tree"][0, 0])
    np.testing.assert_array_equal(out[0, 1], w["v_tree"][0, 0])

    w = _wl(rng, [7, 5], [20, 33], n_q=2, n_kv=1, d=16, page_size=16)
    c = rng.standard_normal(16).astype(np.float32)
    w["v_cache"][:] = c
    w["v_tree"][:] = c
    out, _ = _run(w)
    np.testing.assert_allclose(out, np.broadcast_to(c, out.shape), rtol=1e-7, atol=0)

    w = _wl(rng, [6], [10], n_q=1, n_kv=1, d=8, page_size=16)
    w["k_cache"][:] = 0.5
    w["k_tree"][:] = 0.5
    out, _ = _run(w)
    par = w["tree_parent"]
    kp, vp = _dense_prefix(w, 0, 0)
    for j in range(6):
        anc, u = [], j
        while True:
            anc.append(u)
            if u == 0:
                break
            u = par[u]
        rows = np.vstack([vp, w["v_tree"][anc, 0].astype(np.float64)])
        np.testing.assert_allclose(out[j, 0], rows.mean(0), atol=1e-6)


def test_page_permutation_and_gqa_bitexact():
    """Physical page placement is irrelevant; GQA equals MHA with replicated KV heads."""
    rng = np.random.default_rng(4)
    w = _wl(rng, [5, 8], [40, 70], n_q=4, n_kv=2, d=32, page_size=16)
    out, lse = _run(w)
    perm = rng.permutation(w["k_cache"].shape[0])
    inv = np.argsort(perm)
    w2 = dict(w)
    w2["k_cache"] = w["k_cache"][perm]
    w2["v_cache"] = w["v_cache"][perm]
    w2["page_table"] = np.where(w["page_table"] >= 0, inv[np.maximum(w["page_table"], 0)], -1).astype(np.int32)
    out2, lse2 = _run(w2)
    np.testing.assert_array_equal(out, out2)
    w3 = dict(w)
    w3["k_cache"] = np.repeat(w["k_cache"], 2, axis=1)
    w3["v_cache"] = np.repeat(w["v_cache"], 2, axis=1)
    w3["k_tree"] = np.repeat(w["k_tree"], 2, axis=1)
    w3["v_tree"] = np.repeat(w["v_tree"], 2, axis=1)
    out3, _ = _run(w3)
    np.testing.assert_array_equal(out, out3)


def test_star_tree_sibling_permutation():
    """P-att-5: in a star, row j sees prefix + {root, j}; permuting siblings permutes rows."""
    rng = np.random.default_rng(6)
    w = _wl(rng, [6], [25], n_q=2, n_kv=1, d=16, page_size=16, shape="star")
    out, _ = _run(w)
    perm = np.concatenate([[0], 1 + rng.permutation(5)])
    w2 = dict(w)
    for key in ("q", "k_tree", "v_tree"):
        w2[key] = w[key][perm]
    out2, _ = _run(w2)
    np.testing.assert_array_equal(out2, out[perm])
