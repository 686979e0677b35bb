"""Pins of the NEXT-3(b) oracle (oracle/mss.py, reading R25): SpecInfer
multi-step speculative sampling is LOSSLESS -- whatever the draft, the tokens
it emits are distributed as the target model's.  These tests check the oracle
against that property (chi-squared), against the single-draft closed form
sum_x min(p, q) (Leviathan et al. / Chen et al.), and show the test has power
(a mutant without the residual update fails it).  CPU only."""
import numpy as np
import pytest
from scipy import stats

import oracle
from oracle import mss

V = 5


def _dist(rng, sharp):
    z = rng.normal(0.0, sharp, V)
    e = np.exp(z - z.max())
    return (e / e.sum()).astype(np.float32)


def _norm(d):
    d = np.asarray(d, np.float64)
    return d / d.sum()


def _toy_models(seed):
    """A 2-level toy draft model q(.|ctx) and target model p(.|ctx) over V tokens."""
    rng = np.random.default_rng(seed)
    q = {(): _dist(rng, 1.5)}
    p = {(): _dist(rng, 1.5)}
    for a in range(V):
        q[(a,)] = _dist(rng, 1.5)
        p[(a,)] = _dist(rng, 1.5)
        for b in range(V):
            p[(a, b)] = _dist(rng, 1.0)
    return q, p


def _trial(rng, q, p, k1, k2, node_fn=None):
    """One speculation + MSS verification of a 2-level tree whose children are
    drawn i.i.d. from the draft (SpecInfer's stochastic speculation).  Returns
    the emitted token sequence (accepted drafts, then the bonus)."""
    toks, par, ctx = [0], [0], [()]
    for _ in range(k1):
        toks.append(int(rng.choice(V, p=_norm(q[()]))))
        par.append(0)
        ctx.append((toks[-1],))
    for c in range(1, k1 + 1):
        a = toks[c]
        for _ in range(k2):
            toks.append(int(rng.choice(V, p=_norm(q[(a,)]))))
            par.append(c)
            ctx.append((a, toks[-1]))
    K = len(toks)
    P = np.stack([p[cx] for cx in ctx])
    Q = np.stack([q[cx] if cx in q else np.zeros(V, np.float32) for cx in ctx])
    r = rng.random(K).astype(np.float32)
    r = np.where(r == 0, np.float32(1.0), r)
    rb = rng.random(K).astype(np.float32)
    rb = np.where(rb == 0, np.float32(1.0), rb)
    if node_fn is None:
        emit, _ = mss.mss_tokens(np.array([0, K]), np.array(par), np.array(toks), P, Q, r, rb)
    else:
        emit = np.array([node_fn(P[u], Q[u], [toks[c] for c in range(K) if par[c] == u and c > u],
                                 [r[c] for c in range(K) if par[c] == u and c > u], rb[u]) for u in range(K)])
    w = oracle.accept_walk(np.array([0, K], np.int32), np.array(par, np.int32), np.array(toks, np.int32),
                           target_tokens=emit.astype(np.int32), max_path=4)
    L = int(w["accept_len"][0])
    path = [int(x) for x in w["accept_path"][0][:L]]
    return [toks[v] for v in path[1:]] + [int(w["bonus_token"][0])]


def _chi2_p(counts, probs):
    probs = np.asarray(probs, np.float64)
    probs = probs / probs.sum()
    n = counts.sum()
    exp = probs * n
    keep = exp > 0
    return stats.chisquare(counts[keep], exp[keep] * counts[keep].sum() / exp[keep].sum()).pvalue


@pytest.mark.parametrize("seed,k1,k2", [(1, 3, 2), (2, 1, 1), (3, 4, 3)])
def test_mss_is_lossless(seed, k1, k2):
    q, p = _toy_models(seed)
    rng = np.random.default_rng(100 + seed)
    n = 12000
    first = np.zeros(V, np.int64)
    second = {}
    for _ in range(n):
        seq = _trial(rng, q, p, k1, k2)
        first[seq[0]] += 1
        if len(seq) >= 2:
            second.setdefault(seq[0], np.zeros(V, np.int64))[seq[1]] += 1
    assert _chi2_p(first, p[()]) > 1e-3, first
    a = max(second, key=lambda k: second[k].sum())
    assert second[a].sum() > 300
    assert _chi2_p(second[a], p[(a,)]) > 1e-3, (a, second[a])


def test_single_draft_acceptance_rate_closed_form():
    """One child drawn from q: P(accept) = sum_x min(p(x), q(x))."""
    q, p = _toy_models(7)
    rng = np.random.default_rng(8)
    n = 20000
    acc = 0
    for _ in range(n):
        x = int(rng.choice(V, p=_norm(q[()])))
        r = np.float32(max(rng.random(), 1e-7))
        tok, j, _ = mss.mss_node(p[()], q[()], [x], [r], np.float32(0.5))
        acc += j == 0
    want = float(np.minimum(p[()].astype(np.float64), q[()].astype(np.float64)).sum())
    se = np.sqrt(want * (1 - want) / n)
    assert abs(acc / n - want) < 4 * se, (acc / n, want)


def test_mutant_without_residual_fails_chi2():
    """Power: retrying every child against the unchanged target (no residual
    update) over-emits draft-likely tokens; the same chi-squared test rejects it."""
    def naive(pr, qr, kids, rs, rb):
        pr = pr.astype(np.float64)
        qr = qr.astype(np.float64)
        for x, r in zip(kids, rs):
            if r * qr[x] <= pr[x]:
                return x
        c = np.cumsum(pr)
        return int(np.searchsorted(c, rb * c[-1]))
    q, p = _toy_models(1)
    # a draft far from the target makes the bias large
    q[()] = np.roll(p[()], 2)
    rng = np.random.default_rng(5)
    first = np.zeros(V, np.int64)
    for _ in range(8000):
        first[_trial(rng, q, p, 3, 1, node_fn=naive)[0]] += 1
    assert _chi2_p(first, p[()]) < 1e-6, first


def test_emitted_token_identifies_accepted_child():
    """A rejected token gets zero residual mass: an earlier sibling with the
    same token can never shadow the accepted child, and the bonus is never a
    tried child's token (so the token walk is the MSS walk)."""
    rng = np.random.default_rng(9)
    q, p = _toy_models(4)
    for _ in range(3000):
        kids = [int(x) for x in rng.choice(V, size=4, p=_norm(q[()]))]
        r = [np.float32(max(rng.random(), 1e-7)) for _ in kids]
        tok, j, _ = mss.mss_node(p[()], q[()], kids, r, np.float32(max(rng.random(), 1e-7)))
        if j >= 0:
            assert kids.index(tok) == j
        else:
            assert tok not in kids


def test_mss_walk_equals_token_walk_on_emitted_tokens():
    """mss_walk (accepted-child indices) and the greedy token walk over the
    per-node emitted tokens (R13) give the same path and bonus: the emitted
    token identifies the accepted child (R25)."""
    rng = np.random.default_rng(21)
    q, p = _toy_models(5)
    for _ in range(300):
        k1, k2 = int(rng.integers(1, 4)), int(rng.integers(0, 3))
        toks, par, ctx = [0], [0], [()]
        for _ in range(k1):
            toks.append(int(rng.choice(V, p=_norm(q[()]))))
            par.append(0)
            ctx.append((toks[-1],))
        for c in range(1, k1 + 1):
            for _ in range(k2):
                toks.append(int(rng.choice(V, p=_norm(q[(toks[c],)]))))
                par.append(c)
                ctx.append((toks[c], toks[-1]))
        K = len(toks)
        P = np.stack([p[cx] for cx in ctx])
        Q = np.stack([q[cx] if cx in q else np.zeros(V, np.float32) for cx in ctx])
        r = np.maximum(rng.random(K), 1e-7).astype(np.float32)
        rb = np.maximum(rng.random(K), 1e-7).astype(np.float32)
        off = np.array([0, K], np.int32)
        emit, _ = mss.mss_tokens(off, np.array(par), np.array(toks), P, Q, r, rb)
        w = oracle.accept_walk(off, np.array(par, np.int32), np.array(toks, np.int32),
                               target_tokens=emit.astype(np.int32), max_path=4)
        m = mss.mss_walk(off, np.array(par), np.array(toks), P, Q, r, rb, 4)
        assert int(m["accept_len"][0]) == int(w["accept_len"][0])
        assert int(m["bonus_token"][0]) == int(w["bonus_token"][0])
        assert np.array_equal(m["accept_path"][0], w["accept_path"][0])
