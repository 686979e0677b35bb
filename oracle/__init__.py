"""CPU oracle for the AdaServe select -> verify -> accept hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2501_12162_b200`` (the CUDA product
path) and neither imports the other; the only shared module is the seeded
input generator ``synth`` (which holds none of the method's arithmetic).

Contents
--------
* ``select_literal``  -- Alg. 2 step by step, in C
  (``adaserve_ref.c``), the reference the GPU select is compared to bit-exactly.
* ``select_closed_form`` -- O2: the data-parallel restatement of Alg. 2
  (per-request sorted prefixes, clamped scan in A order, global top-R).  Pinned
  to ``select_literal`` by fuzzing (proof sketch in DESIGN.md §Select).
* ``select_per_request_greedy`` / ``equal_greedy_caps`` -- NEXT-4 selection
  variants without SLO awareness: EqualGreedy and Eagle-2 top-m
  (P:L1218), per-request GetTop loops (reading R24); pinned by np.lexsort
  per-request top-k and by the n = 1 identity with GlobalGreedy.
* ``alg1_optimal`` / ``brute_force_optimal`` -- Alg. 1 and an
  exhaustive enumerator; pins App. C optimality on tiny forests.
* ``tree_attn`` -- explicit-mask attention per tree node in fp64 (C).
* ``accept_walk`` / ``commit`` -- the sequential acceptance walk and KV commit (C).
* ``expected_accept_exact`` -- Thm. 1 by exhaustive enumeration of
  per-node target samples, in exact rationals.
* ``beam_step`` / ``beam_search`` -- Step 1 speculation: one
  beam layer = the top-w of the w x |V| expansions by approximated path
  probability f-hat = fl32(f-hat(parent) * M_q(token | X, Path(parent)))
  (P:L691-694), ties (parent asc, token asc) (R8); pinned by exhaustive
  enumeration, the complete-tree case and Thm. 2 containment.

* ``sampling.sample_rows`` -- NEXT-3(a): per-node target samples by
  Gumbel-max with a counter-based generator and a fixed fp32 logarithm
  (reading R23), pinned by the Philox known-answer vectors, the fp64 log and a
  chi-squared test of the Gumbel-max theorem (``tests/test_oracle_sampling.py``).

Parity unpinned: none (see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "adaserve_ref.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

REF_OK = 0
REF_ERR_INVALID_ARG = 1
REF_ERR_BUDGET_TOO_SMALL = 2
REF_ERR_PRECONDITION = 6


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------------------
# Select
# ---------------------------------------------------------------------------
def select_literal(cand_offsets, cand_parent, cand_prob, slo_deficit, depth_d, n_max, budget):
    """Alg. 2 literally (C).  Returns dict(tree_offsets, tree_parent, tree_src,
    tree_depth, slo_count) or raises ValueError on B < n (R10)."""
    lib = _load()
    co = _i32(cand_offsets)
    cp = _i32(cand_parent)
    cf = _f32(cand_prob)
    A = np.ascontiguousarray(slo_deficit, dtype=np.float64)
    n = len(co) - 1
    cap = max(int(budget), 1)
    to = np.zeros(n + 1, np.int32)
    tp = np.full(cap, -7, np.int32)
    ts = np.full(cap, -7, np.int32)
    td = np.full(cap, -7, np.int32)
    sc = np.zeros(max(n, 1), np.int32)
    st = lib.asref_select_literal(ctypes.c_int(n), _p(co), _p(cp), _p(cf), _p(A),
                                  ctypes.c_int(depth_d), ctypes.c_int(n_max), ctypes.c_int(budget),
                                  _p(to), _p(tp), _p(ts), _p(td), _p(sc))
    if st == REF_ERR_BUDGET_TOO_SMALL:
        raise ValueError("budget < n_req (R10)")
    if st != REF_OK:
        raise ValueError(f"oracle select failed: {st}")
    used = int(to[n])
    return dict(tree_offsets=to, tree_parent=tp[:used].copy(), tree_src=ts[:used].copy(),
                tree_depth=td[:used].copy(), slo_count=sc[:n].copy())


def select_closed_form(cand_offsets, cand_parent, cand_prob, slo_deficit, depth_d, n_max, budget):
    """O2: Alg. 2 restated as (1) per-request sort, (2) per-request SLO prefix
    length, (3) clamped exclusive scan in A order, (4) global top-R.  Step
    numbering follows DESIGN.md §Select; each step is the closed form of one
    loop of Alg. 2."""
    co = np.asarray(cand_offsets, np.int64)
    cf = np.asarray(cand_prob, np.float32)
    A = np.asarray(slo_deficit, np.float64)
    n = len(co) - 1
    if budget < n:
        raise ValueError("budget < n_req (R10)")
    B0 = budget - n
    # (1) pi_i: non-root candidates sorted by (f desc, idx asc)  [R8]
    pis = []
    for i in range(n):
        idx = np.arange(1, co[i + 1] - co[i])
        f = cf[co[i] + idx]
        order = np.lexsort((idx, -f.astype(np.float64)))
        pis.append(idx[order])
    # (2) desired_i = min(k*, n_max, C_i - 1), k* = first k with 1 + sum_{t<k} f >= A_cap
    desired = np.zeros(n, np.int64)
    for i in range(n):
        a_cap = min(A[i], depth_d + 1.0)
        acc = 1.0
        k = 0
        lim = min(n_max, len(pis[i]))
        while k < lim and acc < a_cap:
            acc += float(cf[co[i] + pis[i][k]])
            k += 1
        desired[i] = k
    # (3) clamped scan in (A desc, id asc) order
    order = sorted(range(n), key=lambda i: (-A[i], i))
    s = np.zeros(n, np.int64)
    cum = 0
    for i in order:
        s[i] = max(0, min(B0 - cum, desired[i]))
        cum += desired[i]
    # (4) global top-R of the tails under (f desc, req asc, idx asc)
    tails = [(float(cf[co[i] + j]), i, int(j)) for i in range(n) for j in pis[i][s[i]:]]
    R = min(B0 - int(s.sum()), len(tails))
    tails.sort(key=lambda t: (-t[0], t[1], t[2]))
    m = np.zeros(n, np.int64)
    for (_, i, _) in tails[:R]:
        m[i] += 1
    chosen = [set(pis[i][: s[i] + m[i]].tolist()) | {0} for i in range(n)]
    return chosen, s, m


def select_per_request_greedy(cand_offsets, cand_parent, cand_prob, caps):
    """Selection without SLO awareness (NEXT-4, reading R24): request i keeps
    its root and then, caps[i] times or until its candidates run out, GetTop of
    its own remaining candidates -- the linear-scan argmax of (f-hat, -index)
    (R8), as Alg. 2's GetTop restricted to one request.  EqualGreedy
    ("evenly distributes the budget among requests and greedily selects
    tokens from the candidate token tree for each request") uses
    caps = equal_greedy_caps(n, B); Eagle-2's top-m uses caps = m.
    Emitted like select_literal: ascending local index, compact parents, depth;
    'kept' = the non-root nodes taken per request."""
    co = [int(x) for x in cand_offsets]
    n = len(co) - 1
    par = np.asarray(cand_parent, np.int64)
    f = np.asarray(cand_prob, np.float32)
    to = [0]
    tp, ts, td, kept = [], [], [], []
    for i in range(n):
        C = co[i + 1] - co[i]
        chosen = {0}
        for _ in range(int(caps[i])):
            best = None
            for j in range(1, C):  # GetTop: largest f-hat, lowest index on ties
                if j in chosen:
                    continue
                if best is None or f[co[i] + j] > f[co[i] + best]:
                    best = j
            if best is None:
                break
            chosen.add(best)
        nodes = sorted(chosen)
        remap = {v: k for k, v in enumerate(nodes)}
        for v in nodes:
            pv = int(par[co[i] + v]) if v > 0 else 0
            if pv not in remap:
                raise ValueError("selection not ancestor-closed")
            d, u = 0, v
            while u != 0:
                u = int(par[co[i] + u])
                d += 1
            ts.append(v)
            tp.append(remap[pv])
            td.append(d)
        kept.append(len(nodes) - 1)
        to.append(to[-1] + len(nodes))
    return dict(tree_offsets=np.array(to, np.int32), tree_parent=np.array(tp, np.int32),
                tree_src=np.array(ts, np.int32), tree_depth=np.array(td, np.int32), kept=np.array(kept, np.int32))


def equal_greedy_caps(n, budget):
    """EqualGreedy's even split of the budget B (roots included, R1): floor(B/n)
    nodes per request and one more for the first B mod n requests (R24), i.e.
    share - 1 non-root candidates each."""
    if budget < n:
        raise ValueError("budget < n_req (R10)")
    return np.array([budget // n + (1 if i < budget % n else 0) - 1 for i in range(n)], np.int64)


def trees_from_result(res, n):
    """Selected local-index sets per request from a select_literal-style dict."""
    to, ts = res["tree_offsets"], res["tree_src"]
    return [set(ts[to[i]:to[i + 1]].tolist()) for i in range(n)]


def _forest_lists(cand_offsets, cand_parent, cand_prob):
    co = list(map(int, cand_offsets))
    n = len(co) - 1
    par = [list(map(int, cand_parent[co[i]:co[i + 1]])) for i in range(n)]
    prob = [[float(x) for x in cand_prob[co[i]:co[i + 1]]] for i in range(n)]
    return n, par, prob


def alg1_optimal(cand_offsets, cand_parent, cand_prob, slo_deficit, budget):
    """Alg. 1 on a finite forest whose f are the TRUE path
    probabilities.  Readings: R1 (roots charged), R2 (strict budget guard),
    Step 1 in input order (as written), GetTop by (f desc, idx asc) /
    (f desc, req asc, idx asc) (R8).  Running out of candidates in Step 1 on a
    finite forest is INVALID (T_inf is infinite in the paper).
    Returns (list of selected local-index sets, objective) or None (INVALID)."""
    n, par, prob = _forest_lists(cand_offsets, cand_parent, cand_prob)
    B = budget - n
    if B < 0:
        return None
    sel = [{0} for _ in range(n)]
    nacc = [1.0] * n
    for i in range(n):  # Step 1
        while nacc[i] < slo_deficit[i]:
            if B <= 0:
                return None
            cands = [(-prob[i][j], j) for j in range(1, len(prob[i])) if j not in sel[i]]
            if not cands:
                return None
            _, v = min(cands)
            sel[i].add(v)
            nacc[i] += prob[i][v]
            B -= 1
    while B > 0:  # Step 2
        cands = [(-prob[i][j], i, j) for i in range(n) for j in range(1, len(prob[i])) if j not in sel[i]]
        if not cands:
            break
        _, i, v = min(cands)
        sel[i].add(v)
        B -= 1
    obj = sum(Fraction(prob[i][j]) for i in range(n) for j in sel[i])
    return sel, obj


def _closed_subsets(par):
    """All root-containing ancestor-closed subsets of one tree (as frozensets)."""
    K = len(par)
    out = []
    for mask in range(1 << (K - 1)):
        s = {0} | {j for j in range(1, K) if mask >> (j - 1) & 1}
        if all(par[j] in s for j in s if j != 0):
            out.append(frozenset(s))
    return out


def brute_force_optimal(cand_offsets, cand_parent, cand_prob, slo_deficit, budget):
    """Exhaustive enumeration: over all families of root-containing connected
    subtrees with sum |T_i| <= B and sum_{v in T_i} f(v) >= A_i for every i
    (Eq. 1 and Eq. 4), maximise sum f.  Exact
    rational arithmetic.  Returns (best objective, one optimal family) or None."""
    n, par, prob = _forest_lists(cand_offsets, cand_parent, cand_prob)
    per = []
    for i in range(n):
        opts = []
        for s in _closed_subsets(par[i]):
            val = sum(Fraction(prob[i][j]) for j in s)
            if val >= Fraction(slo_deficit[i]):
                opts.append((len(s), val, s))
        per.append(opts)
    best = None
    for combo in itertools.product(*per):
        size = sum(c[0] for c in combo)
        if size > budget:
            continue
        val = sum(c[1] for c in combo)
        if best is None or val > best[0]:
            best = (val, [set(c[2]) for c in combo])
    return best


# ---------------------------------------------------------------------------
# Speculation (Step 1): beam search over the draft model's distributions
# ---------------------------------------------------------------------------
def beam_step(probs, f_parent, width):
    """One beam layer for ONE request.  probs [w_in, V] fp32:
    the draft conditional M_q(token | X, Path(parent)) of every kept node of the
    previous layer (rows in rank order); f_parent [w_in] fp32 their f-hat.
    Every expansion (parent k, token t) gets f-hat = fl32(f_parent[k] *
    probs[k, t]) (the product of conditionals along the path);
    the layer keeps the `width` largest by (f-hat desc, parent asc, token asc)
    (R8; "the w with the highest approximated path probabilities").
    Returns (parent_rank [width], token [width], f-hat [width]) in rank order."""
    probs = np.asarray(probs, np.float32)
    f_parent = np.asarray(f_parent, np.float32)
    w_in, V = probs.shape
    f = (f_parent[:, None] * probs).astype(np.float32)        # fp32 products
    par = np.repeat(np.arange(w_in), V)
    tok = np.tile(np.arange(V), w_in)
    ff = f.reshape(-1)
    order = np.lexsort((tok, par, -ff.astype(np.float64)))[:width]
    return par[order].astype(np.int32), tok[order].astype(np.int32), ff[order].astype(np.float32)


def beam_search(root_probs_fn, depth, width):
    """Step 1 for one request: d beam layers.  root_probs_fn(path)
    returns the draft distribution [V] after the token path `path` (a tuple of
    token ids from the root).  Returns the candidate tree in the forest layout
    the select kernel consumes: node 0 = root (f-hat 1), then layer by layer in
    rank order -- (parent [N], token [N] (root token = -1), prob [N] fp32)."""
    parent, token, prob, paths = [0], [-1], [np.float32(1.0)], [()]
    layer = [0]
    for _ in range(depth):
        probs = np.stack([np.asarray(root_probs_fn(paths[u]), np.float32) for u in layer])
        fpar = np.array([prob[u] for u in layer], np.float32)
        pr, tk, fv = beam_step(probs, fpar, width)
        new = []
        for k in range(len(pr)):
            u = layer[int(pr[k])]
            parent.append(u)
            token.append(int(tk[k]))
            prob.append(np.float32(fv[k]))
            paths.append(paths[u] + (int(tk[k]),))
            new.append(len(parent) - 1)
        layer = new
    return np.array(parent, np.int32), np.array(token, np.int32), np.array(prob, np.float32)


# ---------------------------------------------------------------------------
# Verify
# ---------------------------------------------------------------------------
def tree_attn(q, k_tree, v_tree, k_cache, v_cache, page_table, kv_len, tree_offsets, tree_parent,
              sm_scale, n_threads=1, want_lse=True):
    """Explicit-mask attention per tree node (C, fp64 accumulate, fp32 out).
    Array shapes as in DESIGN.md: q [R, n_q, d], k_tree/v_tree [R, n_kv, d],
    caches [pages, n_kv, page_size, d], page_table [n, max_pages]."""
    lib = _load()
    q = _f32(q)
    kt, vt = _f32(k_tree), _f32(v_tree)
    kc, vc = _f32(k_cache), _f32(v_cache)
    pt = _i32(page_table)
    kl = _i32(kv_len)
    to = _i32(tree_offsets)
    tp = _i32(tree_parent)
    R, n_q, d = q.shape
    n_kv = kt.shape[1]
    page_size = kc.shape[2]
    n = len(to) - 1
    out = np.zeros_like(q)
    lse = np.zeros((R, n_q), np.float32) if want_lse else None
    st = lib.asref_tree_attn(ctypes.c_int(n), ctypes.c_int(n_q), ctypes.c_int(n_kv), ctypes.c_int(d),
                             _p(q), _p(kt), _p(vt), _p(kc), _p(vc), ctypes.c_int(page_size), _p(pt),
                             ctypes.c_int(pt.shape[1]), _p(kl), _p(to), _p(tp),
                             ctypes.c_float(sm_scale), _p(out), _p(lse), ctypes.c_int(n_threads))
    if st != REF_OK:
        raise ValueError(f"oracle attention failed: {st}")
    return out, lse


# ---------------------------------------------------------------------------
# Accept
# ---------------------------------------------------------------------------
def accept_walk(tree_offsets, tree_parent, tree_tokens, target_tokens=None, target_logits=None,
                max_path=16):
    lib = _load()
    to = _i32(tree_offsets)
    tp = _i32(tree_parent)
    tt = _i32(tree_tokens)
    n = len(to) - 1
    tgt = None if target_tokens is None else _i32(target_tokens)
    lg = None if target_logits is None else _f32(target_logits)
    vocab = 0 if lg is None else lg.shape[1]
    al = np.zeros(max(n, 1), np.int32)
    ap = np.zeros((max(n, 1), max_path), np.int32)
    bt = np.zeros(max(n, 1), np.int32)
    st = lib.asref_accept_walk(ctypes.c_int(n), _p(to), _p(tp), _p(tt), _p(tgt), _p(lg),
                               ctypes.c_int(vocab), ctypes.c_int(max_path), _p(al), _p(ap), _p(bt))
    return dict(accept_len=al[:n], accept_path=ap[:n], bonus_token=bt[:n], status=st)


def commit(tree_offsets, accept_len, accept_path, k_tree, v_tree, k_cache, v_cache, page_table, kv_len):
    """In-place byte-exact commit on host copies.  k_tree etc. are numpy arrays
    of a 2- or 4-byte dtype (bf16 data can be passed as uint16)."""
    lib = _load()
    assert k_cache.flags.c_contiguous and v_cache.flags.c_contiguous and kv_len.dtype == np.int32
    to = _i32(tree_offsets)
    al = _i32(accept_len)
    ap = _i32(accept_path)
    pt = _i32(page_table)
    kt = np.ascontiguousarray(k_tree)
    vt = np.ascontiguousarray(v_tree)
    n = len(to) - 1
    n_kv, d = kt.shape[1], kt.shape[2]
    st = lib.asref_commit(ctypes.c_int(n), _p(to), _p(al), _p(ap), ctypes.c_int(ap.shape[1]),
                          _p(kt), _p(vt), ctypes.c_int(kt.itemsize), ctypes.c_int(n_kv), ctypes.c_int(d),
                          _p(k_cache), _p(v_cache), ctypes.c_int(k_cache.shape[2]), _p(pt),
                          ctypes.c_int(pt.shape[1]), _p(kv_len))
    return st


def expected_accept_exact(parent, tokens, cond_dists):
    """Thm. 1 pin (App. A) by brute force.

    parent[j], tokens[j] describe one tree (root 0).  cond_dists[j] is the
    target's conditional distribution at node j over a vocab of size V, as a
    list of Fractions summing to 1.  Enumerate every joint assignment of one
    target sample per node (V^K of them), run the acceptance walk (R13) on
    each, and return (E[accept_len], sum_v f(v)) as exact Fractions, where
    f(v) = product of the target conditionals of the draft tokens on the path
    root -> v (the probability that the walk accepts that path)."""
    K = len(parent)
    V = len(cond_dists[0])
    exp_len = Fraction(0)
    for assign in itertools.product(range(V), repeat=K):
        w = Fraction(1)
        for j in range(K):
            w *= cond_dists[j][assign[j]]
        if w == 0:
            continue
        v, length = 0, 1
        while True:
            t = assign[v]
            nxt = next((c for c in range(v + 1, K) if parent[c] == v and tokens[c] == t), None)
            if nxt is None:
                break
            v, length = nxt, length + 1
        exp_len += w * length
    f = [Fraction(1)] * K
    for j in range(1, K):
        f[j] = f[parent[j]] * cond_dists[parent[j]][tokens[j]]
    return exp_len, sum(f)
