"""CPU pins of the speculation oracle (Step 1 beam search):
Thm. 2 containment against Alg. 1 / brute force, the complete-tree
case (w >= |V|^d), the Fig. 4 shape (d = 3, w = 2 -> 7 nodes), w = 1 == greedy
decoding (argmax at every step), and f-hat monotone along every edge."""
import itertools

import numpy as np
import pytest

import oracle


def _draft(rng, V, sigma=1.5):
    """A random draft model: a fixed fp32 distribution per token path."""
    table = {}

    def probs(path):
        if path not in table:
            z = rng.normal(0.0, sigma, V)
            e = np.exp(z - z.max())
            table[path] = (e / e.sum()).astype(np.float32)
        return table[path]
    return probs


def _complete_tree(probs_fn, V, depth):
    """T_inf truncated at `depth`: every path, f = fl32 product of conditionals
    (drift 0: the approximation is exact).  Returns parent, prob,
    token paths (topological: BFS order)."""
    parent, prob, paths = [0], [np.float32(1.0)], [()]
    frontier = [0]
    for _ in range(depth):
        nxt = []
        for u in frontier:
            q = probs_fn(paths[u])
            for t in range(V):
                parent.append(u)
                prob.append(np.float32(prob[u] * q[t]))
                paths.append(paths[u] + (t,))
                nxt.append(len(parent) - 1)
        frontier = nxt
    return np.array(parent, np.int32), np.array(prob, np.float32), paths


def _depth(par, j):
    d = 0
    while j:
        j = par[j]
        d += 1
    return d


@pytest.mark.parametrize("seed", range(40))
def test_thm2_containment(seed):
    """Thm. 2: the optimal tree T_opt of Alg. 1 (budget B) is a subtree of the
    candidate tree of a D_opt-step beam search with width B."""
    rng = np.random.default_rng(seed)
    V = int(rng.integers(2, 4))
    B = int(rng.integers(2, 6))
    probs_fn = _draft(rng, V)
    par, prob, paths = _complete_tree(probs_fn, V, B - 1)   # |T_opt| <= B: depth <= B - 1
    co = np.array([0, len(par)], np.int32)
    A = [float(rng.uniform(0.0, 1.5))]
    res = oracle.alg1_optimal(co, par, prob, A, B)
    if res is None:
        return
    sel, obj = res
    if len(par) <= 16:  # Alg. 1 is optimal (App. C): cross-check by enumeration where feasible
        bf = oracle.brute_force_optimal(co, par, prob, A, B)
        assert bf is not None and bf[0] == obj
    T = sel[0]
    d_opt = max(_depth(par, j) for j in T)
    bpar, btok, bprob = oracle.beam_search(probs_fn, d_opt, B)
    bpaths = [()]
    for j in range(1, len(bpar)):
        bpaths.append(bpaths[bpar[j]] + (int(btok[j]),))
    assert {paths[j] for j in T} <= set(bpaths)


def test_complete_tree_when_width_covers_every_path():
    rng = np.random.default_rng(1)
    V, d = 3, 3
    probs_fn = _draft(rng, V)
    par, tok, prob = oracle.beam_search(probs_fn, d, V ** d)
    sizes = [sum(1 for j in range(1, len(par)) if _depth(par, j) == k) for k in range(1, d + 1)]
    assert sizes == [V, V ** 2, V ** 3]
    paths = {()}
    for j in range(1, len(par)):
        p = [int(tok[j])]
        u = par[j]
        while u:
            p.append(int(tok[u]))
            u = par[u]
        paths.add(tuple(reversed(p)))
    assert paths == {tuple(x) for k in range(d + 1) for x in itertools.product(range(V), repeat=k)}


def test_fig4_shape():
    """Fig. 4: three speculation steps with beam width 2 give the
    root plus 2 nodes per layer."""
    rng = np.random.default_rng(2)
    par, tok, prob = oracle.beam_search(_draft(rng, 50), 3, 2)
    assert len(par) == 7
    assert [_depth(par, j) for j in range(7)] == [0, 1, 1, 2, 2, 3, 3]


@pytest.mark.parametrize("seed", range(5))
def test_width_one_is_greedy_decoding(seed):
    rng = np.random.default_rng(10 + seed)
    V, d = 40, 6
    probs_fn = _draft(rng, V, sigma=0.7)
    par, tok, prob = oracle.beam_search(probs_fn, d, 1)
    path = ()
    f = np.float32(1.0)
    for k in range(1, d + 1):
        q = probs_fn(path)
        t = int(np.argmax(q))          # textbook greedy step (lowest index on ties)
        f = np.float32(f * q[t])
        path = path + (t,)
        assert int(tok[k]) == t and par[k] == k - 1 and prob[k] == f


def test_fhat_monotone_along_edges():
    rng = np.random.default_rng(3)
    par, tok, prob = oracle.beam_search(_draft(rng, 30, sigma=3.0), 5, 4)
    assert all(prob[j] <= prob[par[j]] for j in range(1, len(par)))
    assert prob[0] == 1.0
