"""Pins of the NEXT-3(a) sampling oracle (oracle/sampling.py, reading R23)
against things other than itself: published known-answer vectors, the fp64
logarithm, exact representability, and the Gumbel-max theorem (the samples
follow softmax(logits * inv_T)) by a chi-squared test."""
import numpy as np
import pytest
from scipy import stats

from oracle import sampling as S


@pytest.mark.parametrize("ctr,key,want", [
    # Random123 kat_vectors, philox4x32 10 rounds
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
])
def test_philox_known_answers(ctr, key, want):
    got = S.philox4x32_10(*[np.uint32(c) for c in ctr], np.uint32(key[0]), np.uint32(key[1]))
    assert [int(g) for g in got] == want


def test_uniform_exact_and_open_interval():
    x = np.array([0, 1 << 9, 0xFFFFFFFF, 0x80000000], np.uint32)
    u = S.uniform_from_bits(x).astype(np.float64)
    want = np.array([1, 3, 2 ** 24 - 1, 2 ** 23 + 1], np.float64) * 2.0 ** -24
    np.testing.assert_array_equal(u, want)
    assert u.min() > 0 and u.max() < 1


def test_ln_f32_against_fp64_log():
    rng = np.random.default_rng(0)
    x = np.concatenate([np.exp(rng.uniform(-80, 80, 400000)), rng.uniform(1e-8, 20, 400000),
                        [1.0, 2.0, 0.5, np.sqrt(2.0), 1 - 2 ** -24, 2 ** -24, 16.63]]).astype(np.float32)
    x = x[(x > 1.2e-38) & np.isfinite(x)]
    ref = np.log(x.astype(np.float64))
    got = S.ln_f32(x).astype(np.float64)
    assert np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))) < 3e-7
    assert S.ln_f32(np.float32(1.0)) == 0.0


def test_gumbel_moments():
    g = S.gumbel(np.arange(40), 4096, seed=11).astype(np.float64).ravel()
    assert abs(g.mean() - np.euler_gamma) < 0.01          # E = Euler-Mascheroni constant
    assert abs(g.std() - np.pi / np.sqrt(6.0)) < 0.01      # sd = pi / sqrt 6


@pytest.mark.parametrize("V,inv_t,seed", [(6, 0.8, 1), (11, 2.5, 2), (3, 0.0, 3)])
def test_gumbel_max_follows_softmax(V, inv_t, seed):
    rng = np.random.default_rng(seed)
    logits = rng.normal(0.0, 1.5, V).astype(np.float32)
    n = 60000
    tok = S.sample_rows(np.broadcast_to(logits, (n, V)), inv_t, seed=1234 + seed)
    counts = np.bincount(tok, minlength=V)
    z = logits.astype(np.float64) * np.float64(np.float32(inv_t))
    p = np.exp(z - z.max())
    p /= p.sum()
    chi2 = float(((counts - n * p) ** 2 / (n * p)).sum())
    assert stats.chi2.sf(chi2, V - 1) > 1e-4, (counts, n * p)


def test_ties_lowest_index_and_rows_independent():
    lg = np.zeros((4, 8), np.float32)
    lg[:, 3] = 1e30  # dominates any Gumbel draw
    assert S.sample_rows(lg, 1.0, seed=5).tolist() == [3, 3, 3, 3]
    lg = np.zeros((2000, 16), np.float32)
    tok = S.sample_rows(lg, 1.0, seed=9)
    assert len(set(tok.tolist())) == 16  # different rows draw different noise
    # the same (seed, offset, row) reproduces; another offset does not
    a = S.sample_rows(lg[:50], 1.0, seed=9, offset=0)
    b = S.sample_rows(lg[:50], 1.0, seed=9, offset=1)
    np.testing.assert_array_equal(a, tok[:50])
    assert (a != b).any()


def test_stochastic_walk_matches_theorem1():
    """Thm. 1 for the sampler + walk pair: with per-node target
    samples from sample_rows and f(v) the product of target conditionals of the
    tokens on v's path, E[accept_len] = sum_v f(v).  Monte Carlo over 40 000
    independent trials (different rows of the Philox stream) of one tree."""
    import oracle
    rng = np.random.default_rng(21)
    V = 4
    parent = np.array([0, 0, 0, 1, 1, 2, 3, 3, 5], np.int32)  # topological, root 0
    token = np.array([0, 0, 1, 2, 3, 1, 0, 2, 3], np.int32)  # siblings distinct
    K = len(parent)
    logits = rng.normal(0.0, 1.2, (K, V)).astype(np.float32)
    p = np.exp(logits.astype(np.float64))
    p /= p.sum(axis=1, keepdims=True)
    f = np.ones(K)
    for c in range(1, K):
        f[c] = f[parent[c]] * p[parent[c], token[c]]
    trials = 40000
    tgt = S.sample_rows(np.tile(logits, (trials, 1)), 1.0, seed=2024)
    offs = np.arange(0, (trials + 1) * K, K, dtype=np.int32)
    w = oracle.accept_walk(offs, np.tile(parent, trials), np.tile(token, trials), target_tokens=tgt, max_path=K + 1)
    al = w["accept_len"].astype(np.float64)
    se = al.std() / np.sqrt(trials)
    assert abs(al.mean() - f.sum()) < 4 * se, (al.mean(), f.sum(), se)
