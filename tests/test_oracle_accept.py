"""Pins for the acceptance walk + commit oracle (O5).

Thm. 1 is checked in exact rationals by enumerating every joint
target-sample assignment on tiny trees; chains reduce to sequence speculative
decoding; Monte Carlo agrees within 3 sigma; commit is byte-exact.
"""
from fractions import Fraction

import numpy as np

import oracle
import synth


def _rand_dist(rng, V):
    w = rng.integers(1, 6, V)
    w[rng.integers(0, V)] = 0 if V > 2 else w[0]
    tot = int(w.sum())
    return [Fraction(int(x), tot) for x in w]


def test_thm1_exact_enumeration():
    """E[accept_len] == sum_{v in T} f(v) exactly (Thm. 1, App. A),
    for trees with distinct sibling tokens and target conditionals over |V|<=3."""
    rng = np.random.default_rng(0)
    for _ in range(120):
        K = int(rng.integers(1, 7))
        V = int(rng.integers(2, 4))
        par = synth.random_tree_parents(rng, K)
        toks = [0] * K
        ok = True
        for p in range(K):
            kids = [c for c in range(1, K) if par[c] == p]
            if len(kids) > V:
                ok = False
                break
            vals = rng.permutation(V)[: len(kids)]
            for c, t in zip(kids, vals):
                toks[c] = int(t)
        if not ok:
            continue
        dists = [_rand_dist(rng, V) for _ in range(K)]
        e, f = oracle.expected_accept_exact(list(par), toks, dists)
        assert e == f
        # the C walk on every assignment reproduces the same enumeration
        import itertools
        assigns = list(itertools.product(range(V), repeat=K))
        n = len(assigns)
        to = np.arange(n + 1, dtype=np.int32) * K
        res = oracle.accept_walk(to, np.tile(par, n), np.tile(toks, n),
                                 target_tokens=np.array(assigns, np.int32).reshape(-1), max_path=K + 1)
        wts = [np.prod([float(dists[j][a[j]]) for j in range(K)]) for a in assigns]
        assert abs(np.dot(wts, res["accept_len"]) - float(f)) < 1e-12


def test_chain_is_sequence_speculative_decoding():
    """P-acc-2: parent[j]=j-1 -> accept_len = 1 + longest k with draft[t]==target[t-1]."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        K = int(rng.integers(1, 12))
        draft = rng.integers(0, 3, K).astype(np.int32)
        tgt = rng.integers(0, 3, K).astype(np.int32)
        res = oracle.accept_walk(np.array([0, K], np.int32), synth.random_tree_parents(rng, K, shape="chain"),
                                 draft, target_tokens=tgt, max_path=K)
        k = 0
        while k + 1 < K and draft[k + 1] == tgt[k]:
            k += 1
        assert res["accept_len"][0] == k + 1
        assert res["bonus_token"][0] == tgt[k]
        assert res["accept_path"][0, : k + 1].tolist() == list(range(k + 1))


def test_degenerate_cases_and_logits():
    """P-acc-3: root-only -> len 1, bonus = root target; greedy logits argmax picks
    the lowest index on ties (R13)."""
    res = oracle.accept_walk(np.array([0, 1], np.int32), [0], [5], target_tokens=[9], max_path=4)
    assert res["accept_len"][0] == 1 and res["bonus_token"][0] == 9
    par = [0, 0, 0, 1]
    toks = [7, 3, 4, 4]
    logits = np.zeros((4, 6), np.float32)
    logits[0, [4, 3]] = 2.0   # tie between 3 and 4 -> 3 wins -> child 1
    logits[1, 4] = 1.0        # -> child 3 (token 4)
    logits[3, 5] = 1.0
    res = oracle.accept_walk(np.array([0, 4], np.int32), par, toks, target_logits=logits, max_path=4)
    assert res["accept_len"][0] == 3 and res["accept_path"][0, :3].tolist() == [0, 1, 3]
    assert res["bonus_token"][0] == 5
    # duplicate sibling tokens: the lower-index child wins (R13)
    res = oracle.accept_walk(np.array([0, 3], np.int32), [0, 0, 0], [0, 2, 2], target_tokens=[2, 0, 1],
                             max_path=3)
    assert res["accept_path"][0, :2].tolist() == [0, 1] and res["bonus_token"][0] == 0


def test_monte_carlo_thm1():
    """mean accept_len over 1e5 sampled targets within 3 sigma of sum f."""
    rng = np.random.default_rng(2)
    V = 4
    K = 7
    par = np.array([0, 0, 0, 1, 1, 2, 4], np.int32)
    toks = np.array([0, 0, 1, 2, 3, 0, 1], np.int32)
    dist = rng.dirichlet(np.ones(V), K)
    f = np.ones(K)
    for j in range(1, K):
        f[j] = f[par[j]] * dist[par[j], toks[j]]
    N = 100000
    samples = np.stack([rng.choice(V, N, p=dist[j]) for j in range(K)], 1).astype(np.int32)
    res = oracle.accept_walk(np.arange(N + 1, dtype=np.int32) * K, np.tile(par, N), np.tile(toks, N),
                             target_tokens=samples.reshape(-1), max_path=K)
    m = res["accept_len"].mean()
    se = res["accept_len"].std() / np.sqrt(N)
    assert abs(m - f.sum()) < 3 * se + 1e-12


def test_commit_byte_exact():
    """P-acc-5: only path rows land at [L, L+len); every other cache byte unchanged."""
    rng = np.random.default_rng(3)
    n, n_kv, d, ps = 3, 2, 8, 4
    sizes = [5, 1, 7]
    to = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    R = int(to[-1])
    kv_len = np.array([3, 0, 8], np.int32)
    table, n_pages = synth.paged_kv(rng, kv_len, ps, extra_slots=8)
    kc = rng.integers(0, 65535, (n_pages, n_kv, ps, d)).astype(np.uint16)
    vc = rng.integers(0, 65535, (n_pages, n_kv, ps, d)).astype(np.uint16)
    kt = rng.integers(0, 65535, (R, n_kv, d)).astype(np.uint16)
    vt = rng.integers(0, 65535, (R, n_kv, d)).astype(np.uint16)
    al = np.array([3, 1, 2], np.int32)
    ap = np.full((n, 6), -1, np.int32)
    ap[0, :3] = [0, 2, 4]
    ap[1, :1] = [0]
    ap[2, :2] = [0, 6]
    kc2, vc2, kl2 = kc.copy(), vc.copy(), kv_len.copy()
    st = oracle.commit(to, al, ap, kt, vt, kc2, vc2, table, kl2)
    assert st == 0
    assert kl2.tolist() == [6, 1, 10]
    touched = np.zeros(kc.shape[:1] + kc.shape[2:3], bool)
    for i in range(n):
        for k in range(al[i]):
            slot = kv_len[i] + k
            pg = table[i, slot // ps]
            np.testing.assert_array_equal(kc2[pg, :, slot % ps], kt[to[i] + ap[i, k]])
            np.testing.assert_array_equal(vc2[pg, :, slot % ps], vt[to[i] + ap[i, k]])
            touched[pg, slot % ps] = True
    np.testing.assert_array_equal(kc2.transpose(0, 2, 1, 3)[~touched], kc.transpose(0, 2, 1, 3)[~touched])
    np.testing.assert_array_equal(vc2.transpose(0, 2, 1, 3)[~touched], vc.transpose(0, 2, 1, 3)[~touched])
