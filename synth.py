"""Seeded synthetic input generators shared by tests, smoke and bench.

This module holds NO arithmetic of the hot path (select / tree attention /
accept); it only fabricates inputs with the shapes and statistics of the
paper's workloads.  Both the CUDA path and the oracle
consume its outputs; it imports neither.

* ``beam_forest``: the speculation step's output (Step 1, which is
  upstream of the hot path and out of scope): per request a depth-d, width-w
  beam over a synthetic vocab, with f-hat = fp32 product of draft conditionals
  (P:L691-694).  Nodes are ordered by layer then beam rank (topological).
* ``slo_mix``: A(r_i) = (l_i + t_spec)/t_TPOT_i - o_i (Eq. 2) drawn
  from the Table-2 SLO categories -- DESIGN.md §Inputs recipe.
* ``random_forest``: random recursive trees with monotone f-hat and forced ties
  (fuzzing the select tie-break rules).
* ``paged_kv``: page table with randomly permuted pages.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 250112162
LLAMA3_VOCAB = 128256


def rng_for(config_index: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + config_index + 1000003 * salt))


def _softmax64(z):
    z = z - z.max()
    e = np.exp(z)
    return e / e.sum()


def beam_forest(rng, n_req, depth, width, sigma_lo=1.0, sigma_hi=4.0, vocab_s=64,
                with_targets=True):
    """Candidate forest of n_req beams: 1 + depth*width nodes each.

    Returns dict with cand_offsets [n+1], cand_parent [N] (local), cand_prob [N]
    (fp32 f-hat), cand_token [N] (token ids in [0, 128256), distinct among
    siblings), cand_target [N] (a target-model sample at every node drawn from
    that node's own conditional distribution -- the lossless "drift 0" target,
    used as per-node target tokens), and cond (list of per-node conditionals).
    """
    offs = [0]
    parents, probs, toks, targets = [], [], [], []
    for _ in range(n_req):
        sigma = rng.uniform(sigma_lo, sigma_hi)
        tok_map = rng.permutation(LLAMA3_VOCAB)[:vocab_s]
        par = [0]
        f = [np.float32(1.0)]
        tk = [int(tok_map[rng.integers(vocab_s)])]
        cond = []
        layer = [0]
        for _layer in range(depth):
            us, ts, fs = [], [], []
            for u in layer:
                q = _softmax64(rng.normal(0.0, sigma, vocab_s)).astype(np.float32)
                while len(cond) <= u:
                    cond.append(None)
                cond[u] = q
                us.append(np.full(vocab_s, u))
                ts.append(np.arange(vocab_s))
                fs.append((np.float32(f[u]) * q).astype(np.float32))  # fp32 product: f(child) <= f(parent)
            us, ts, fs = np.concatenate(us), np.concatenate(ts), np.concatenate(fs)
            # keep the top `width` expansions by (f desc, parent asc, token asc)
            order = np.lexsort((ts, us, -fs.astype(np.float64)))[:width]
            new_layer = []
            for o in order:
                par.append(int(us[o]))
                f.append(np.float32(fs[o]))
                tk.append(int(tok_map[ts[o]]))
                new_layer.append(len(par) - 1)
            layer = new_layer
        for u in range(len(par)):
            while len(cond) <= u:
                cond.append(None)
            if cond[u] is None:
                cond[u] = _softmax64(rng.normal(0.0, sigma, vocab_s)).astype(np.float32)
        if with_targets:
            for u in range(len(par)):
                p = cond[u].astype(np.float64)
                t = rng.choice(vocab_s, p=p / p.sum())
                targets.append(int(tok_map[t]))
        parents += par
        probs += f
        toks += tk
        offs.append(offs[-1] + len(par))
    out = dict(cand_offsets=np.array(offs, np.int32), cand_parent=np.array(parents, np.int32),
               cand_prob=np.array(probs, np.float32), cand_token=np.array(toks, np.int32))
    if with_targets:
        out["cand_target"] = np.array(targets, np.int32)
    return out


def slo_mix(rng, n_req, t_base=0.030, t_spec=0.040, far_frac=0.03):
    """A(r) for the Table-2 mix: copilot 60% (TPOT 1.2x baseline),
    chatbot 20% (50 ms), summarization 20% (150 ms).  A = t_spec/t_TPOT + dev,
    dev = pace deviation in tokens: U(9,20) for `far_frac` of requests (far
    behind, capped at d+1 by the method), U(0.8,1.6) otherwise."""
    cat = rng.choice(3, size=n_req, p=[0.6, 0.2, 0.2])
    tpot = np.where(cat == 0, 1.2 * t_base, np.where(cat == 1, 0.050, 0.150))
    far = rng.random(n_req) < far_frac
    dev = np.where(far, rng.uniform(9.0, 20.0, n_req), rng.uniform(0.8, 1.6, n_req))
    return (t_spec / tpot + dev).astype(np.float64)


def random_forest(rng, n_req, max_nodes, tie_prob=0.0, min_nodes=1):
    """Random recursive trees: node j>0 picks a parent uniformly in [0, j);
    f(j) = fl32(f(parent) * c), c ~ U(0.05, 0.95), or with probability
    tie_prob c in {1/2, 1/4} and siblings copying each other's f (forced exact
    ties).  Returns cand_offsets, cand_parent, cand_prob."""
    offs = [0]
    par_all, f_all = [], []
    for _ in range(n_req):
        K = int(rng.integers(min_nodes, max_nodes + 1))
        par = [0]
        f = [np.float32(1.0)]
        for j in range(1, K):
            p = int(rng.integers(0, j))
            if rng.random() < tie_prob:
                c = np.float32([0.5, 0.25][int(rng.integers(0, 2))])
            else:
                c = np.float32(rng.uniform(0.05, 0.95))
            par.append(p)
            f.append(np.float32(f[p] * c))
        par_all += par
        f_all += f
        offs.append(offs[-1] + K)
    return dict(cand_offsets=np.array(offs, np.int32), cand_parent=np.array(par_all, np.int32),
                cand_prob=np.array(f_all, np.float32))


def random_tree_parents(rng, K, max_depth=None, shape="random"):
    """Parents of one K-node tree in topological order.  shape in
    {random, chain, star}."""
    if shape == "chain":
        return np.array([0] + list(range(K - 1)), np.int32)
    if shape == "star":
        return np.zeros(K, np.int32)
    par = [0]
    depth = [0]
    for j in range(1, K):
        while True:
            p = int(rng.integers(0, j))
            if max_depth is None or depth[p] < max_depth:
                break
        par.append(p)
        depth.append(depth[p] + 1)
    return np.array(par, np.int32)


def paged_kv(rng, kv_len, page_size, extra_slots=0, spare_pages=0, permute=True):
    """Page table for requests with prefix lengths kv_len (plus extra_slots of
    capacity for commits).  Pages are a random permutation of the pool
    (permute=False: each request's pages are contiguous, for experiments)."""
    kv_len = np.asarray(kv_len, np.int64)
    n = len(kv_len)
    pages_per = (kv_len + extra_slots + page_size - 1) // page_size
    max_pages = int(max(1, pages_per.max() if n else 1))
    total = int(pages_per.sum()) + spare_pages
    perm = rng.permutation(max(total, 1)).astype(np.int32) if permute else np.arange(max(total, 1), dtype=np.int32)
    table = np.full((max(n, 1), max_pages), -1, np.int32)
    c = 0
    for i in range(n):
        for p in range(int(pages_per[i])):
            table[i, p] = perm[c]
            c += 1
    return table[:n] if n else table[:0], max(total, 1)


def bf16_round(x):
    """Round fp32 -> bf16 -> fp32 (round-to-nearest-even), numpy only."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def tree_workload(rng, sizes, kv_lens, n_q, n_kv, d, page_size, shape="random", bf16=True,
                  q_scale=1.0, extra_slots=16, max_depth=None):
    """Verify-step inputs for trees of the given sizes (host arrays, fp32
    holding bf16-rounded values when bf16=True)."""
    sizes = np.asarray(sizes, np.int64)
    n = len(sizes)
    offs = np.zeros(n + 1, np.int32)
    offs[1:] = np.cumsum(sizes)
    R = int(offs[-1])
    par = np.zeros(max(R, 1), np.int32)
    for i in range(n):
        par[offs[i]:offs[i + 1]] = random_tree_parents(rng, int(sizes[i]), max_depth, shape)
    par = par[:R]
    table, n_pages = paged_kv(rng, kv_lens, page_size, extra_slots=extra_slots)
    rnd = (lambda *s: bf16_round(rng.standard_normal(s, dtype=np.float32))) if bf16 else \
        (lambda *s: rng.standard_normal(s, dtype=np.float32))
    q = rnd(max(R, 1), n_q, d)[:R] * np.float32(q_scale)
    if bf16:
        q = bf16_round(q)
    return dict(tree_offsets=offs, tree_parent=par, q=q, k_tree=rnd(max(R, 1), n_kv, d)[:R],
                v_tree=rnd(max(R, 1), n_kv, d)[:R], k_cache=rnd(n_pages, n_kv, page_size, d),
                v_cache=rnd(n_pages, n_kv, page_size, d), page_table=table,
                kv_len=np.asarray(kv_lens, np.int32))


def mss_workload(rng, sizes, vocab, sigma_lo=1.0, sigma_hi=4.0, drift=0.5, shape="random", dup_tokens=False):
    """Inputs of NEXT-3(b) (SpecInfer multi-step speculative sampling, R25):
    per node a draft row q = softmax(z), z ~ N(0, sigma^2) over `vocab`, and a
    target row p = softmax(z + drift * N(0, 1)) (a target near the draft, so
    acceptance is neither certain nor rare); every child's draft token is DRAWN
    from its parent's q (SpecInfer's stochastic speculation), by inverse CDF of
    a uniform; the per-child acceptance uniforms and per-node bonus uniforms
    are U(0, 1] fp32.  dup_tokens draws children from a 4-token support (many
    equal siblings).  Softmaxes in fp64, stored fp32."""
    sizes = [int(k) for k in sizes]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    R = int(offs[-1])
    par = np.concatenate([random_tree_parents(rng, k, shape=shape) for k in sizes]).astype(np.int32) if R else \
        np.zeros(0, np.int32)
    sig = rng.uniform(sigma_lo, sigma_hi, R)
    z = rng.normal(0.0, 1.0, (R, vocab)) * sig[:, None]
    def rows_softmax(x):
        e = np.exp(x - x.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)
    q = rows_softmax(z)
    p = rows_softmax(z + drift * rng.normal(0.0, 1.0, (R, vocab)))
    q32, p32 = q.astype(np.float32), p.astype(np.float32)
    tok = np.zeros(R, np.int32)
    for i, k in enumerate(sizes):
        o = offs[i]
        for j in range(1, k):
            row = q[o + par[o + j]]
            if dup_tokens:
                row = row[:4] / row[:4].sum()
            tok[o + j] = min(int(np.searchsorted(np.cumsum(row), rng.random() * row.sum())), len(row) - 1)
    uni = rng.random(R).astype(np.float32)
    uni[uni == 0] = 1.0
    bon = rng.random(R).astype(np.float32)
    bon[bon == 0] = 1.0
    return {"tree_offsets": offs, "tree_parent": par, "tree_tokens": tok, "p": p32, "q": q32, "uni": uni,
            "bonus_uni": bon}
