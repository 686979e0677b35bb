"""Pins for the select oracle (Alg. 2 literal, O2 closed form, Alg. 1, brute force).

Each pin ties the oracle to something other than itself: the paper's worked
example (Fig. 4), App. C's optimality theorem via exhaustive enumeration, the
closed-form restatement, and library routines (np.lexsort) on special cases.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _forest_from_lists(reqs):
    offs = [0]
    par, prob = [], []
    for r in reqs:
        par += r["parent"]
        prob += r["prob"]
        offs.append(offs[-1] + len(r["parent"]))
    return np.array(offs, np.int32), np.array(par, np.int32), np.array(prob, np.float32)


def test_fig4_golden():
    """P:L602-613 (fig:alg caption)."""
    g = json.load(open(os.path.join(GOLD, "fig4.json")))
    co, cp, cf = _forest_from_lists(g["requests"])
    res = oracle.select_literal(co, cp, cf, g["slo_deficit"], g["depth_d"], g["n_max"], g["budget"])
    names = [r["nodes"] for r in g["requests"]]
    got = [sorted(names[i][j] for j in s) for i, s in enumerate(oracle.trees_from_result(res, 2))]
    assert got == [sorted(t) for t in g["expected"]["trees"]]
    assert res["slo_count"].tolist() == g["expected"]["slo_count"]
    assert int(res["tree_offsets"][-1]) == g["expected"]["used"]
    # compact parents: T0 = root, t1, t3, t5 -> parents 0, 0, 1, 2 ; T1 = root,t1,t2,t3 -> 0,0,0,1
    assert res["tree_parent"].tolist() == [0, 0, 1, 2, 0, 0, 0, 1]
    assert res["tree_depth"].tolist() == [0, 1, 2, 3, 0, 1, 1, 2]
    chosen, s, m = oracle.select_closed_form(co, cp, cf, g["slo_deficit"], g["depth_d"], g["n_max"], g["budget"])
    assert s.tolist() == [1, 2] and m.tolist() == [2, 1]


def test_spec_alg1_examples():
    """S:L236-238 worked examples for Alg. 1."""
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    t = g["alg1_tiny"]
    co = np.array([0, len(t["parent"])], np.int32)
    res = oracle.alg1_optimal(co, t["parent"], np.array(t["prob"], np.float32), t["A"], t["budget"])
    sel, obj = res
    assert sorted(sel[0]) == t["selected"]
    assert abs(float(obj) - t["objective"]) < 1e-6
    bf = oracle.brute_force_optimal(co, t["parent"], np.array(t["prob"], np.float32), t["A"], t["budget"])
    assert bf[0] == obj
    inv = g["alg1_invalid"]
    co2 = np.array([0, 4, 8], np.int32)
    par2 = np.array([0, 0, 0, 0] * 2, np.int32)
    prob2 = np.array([1, .9, .8, .7] * 2, np.float32)
    assert oracle.alg1_optimal(co2, par2, prob2, inv["A"], inv["budget"]) is None
    assert oracle.brute_force_optimal(co2, par2, prob2, inv["A"], inv["budget"]) is None


def test_spec_slo_deficit_values():
    """Eq. 2 rewritten: A = (l + t_spec)/t_TPOT - o."""
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in g["slo_deficit"]:
        assert abs((e["l"] + e["t_spec"]) / e["tpot"] - e["o"] - e["A"]) < 1e-12


def _check_invariants(co, cp, cf, A, d, n_max, B, res):
    n = len(co) - 1
    to, tp, ts = res["tree_offsets"], res["tree_parent"], res["tree_src"]
    assert to[0] == 0 and to[-1] <= B  # Eq. 1
    for i in range(n):
        src = ts[to[i]:to[i + 1]]
        assert src[0] == 0 and np.all(np.diff(src) > 0)  # root first, ascending (topological)
        sset = set(src.tolist())
        for k, j in enumerate(src):
            if j == 0:
                assert tp[to[i] + k] == 0
                continue
            pj = int(cp[co[i] + j])
            assert pj in sset  # ancestor-closed (App. B)
            assert src[tp[to[i] + k]] == pj  # compact parent remap
        assert res["slo_count"][i] <= n_max  # R6


@pytest.mark.parametrize("tie_prob", [0.0, 0.5])
def test_literal_equals_closed_form_fuzz(tie_prob):
    """O1 == O2 on random forests incl. forced exact ties (DESIGN.md proof sketch)."""
    rng = np.random.default_rng(7 + int(tie_prob * 10))
    for it in range(1500):
        n = int(rng.integers(1, 7))
        F = synth.random_forest(rng, n, int(rng.integers(1, 14)), tie_prob=tie_prob)
        co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
        A = rng.uniform(-1, 6, n)
        if rng.random() < 0.3:
            A[rng.integers(0, n)] = A[0]  # equal A -> id tie-break
        d = int(rng.integers(1, 6))
        n_max = int(rng.integers(0, 8))
        B = int(rng.integers(n, co[-1] + 3))
        res = oracle.select_literal(co, cp, cf, A, d, n_max, B)
        _check_invariants(co, cp, cf, A, d, n_max, B, res)
        chosen, s, m = oracle.select_closed_form(co, cp, cf, A, d, n_max, B)
        got = oracle.trees_from_result(res, n)
        assert got == chosen, (it, got, chosen)
        assert res["slo_count"].tolist() == s.tolist()


def test_enumeration_optimality():
    """App. C: Alg. 1's objective == brute-force optimum and
    INVALID <=> infeasible, on every random forest with <= 8 nodes in total;
    and Alg. 2 (literal) == Alg. 1 when its extra knobs are slack."""
    rng = np.random.default_rng(11)
    n_valid = 0
    for it in range(400):
        n = int(rng.integers(1, 4))
        F = synth.random_forest(rng, n, 8 // n, tie_prob=0.0)
        co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
        if co[-1] > 8:
            continue
        A = rng.uniform(0.0, 2.5, n)
        B = int(rng.integers(n, co[-1] + 2))
        a1 = oracle.alg1_optimal(co, cp, cf, A, B)
        bf = oracle.brute_force_optimal(co, cp, cf, A, B)
        assert (a1 is None) == (bf is None), it
        if a1 is None:
            continue
        n_valid += 1
        assert a1[1] == bf[0], it
        d = 64  # A_cap = A
        res = oracle.select_literal(co, cp, cf, A, d, 1000, B)
        assert oracle.trees_from_result(res, n) == [set(s) for s in a1[0]], it
    assert n_valid >= 50


def test_greedy_maximality_lemma():
    """App. C Lemma 'Maximality Under a Fixed Budget': the greedy
    k-node tree (n=1, A<=1 => throughput stage only) has maximal sum f over all
    k-node ancestor-closed subsets."""
    rng = np.random.default_rng(5)
    for _ in range(150):
        F = synth.random_forest(rng, 1, 9, min_nodes=2)
        co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
        K = int(co[-1])
        for k in range(1, K + 1):
            res = oracle.select_literal(co, cp, cf, [0.5], 3, 0, k)
            got = sum(float(cf[j]) for j in oracle.trees_from_result(res, 1)[0])
            best = max(sum(float(cf[j]) for j in s) for s in oracle._closed_subsets(list(cp)) if len(s) == k)
            assert abs(got - best) <= 1e-6 * best


def test_special_cases_library_routines():
    """P-sel-4: reductions of Alg. 2 to np.lexsort top-k (GlobalGreedy P:L1145)."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 6))
        F = synth.random_forest(rng, n, 12, tie_prob=0.3)
        co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
        N = int(co[-1])
        req = np.repeat(np.arange(n), np.diff(co))
        loc = np.arange(N) - co[req]
        nonroot = loc > 0
        # all A <= 1 -> SLO stage inert -> global top-(B-n) by (f desc, req asc, idx asc)
        B = int(rng.integers(n, N + 2))
        res = oracle.select_literal(co, cp, cf, rng.uniform(-2, 1.0, n), 4, 5, B)
        idx = np.nonzero(nonroot)[0]
        order = idx[np.lexsort((loc[idx], req[idx], -cf[idx].astype(np.float64)))][: B - n]
        want = [set([0]) for _ in range(n)]
        for g in order:
            want[req[g]].add(int(loc[g]))
        assert oracle.trees_from_result(res, n) == want
        assert res["slo_count"].tolist() == [0] * n
        # n_max = 0 -> throughput stage only, whatever A is
        res0 = oracle.select_literal(co, cp, cf, rng.uniform(0, 9, n), 8, 0, B)
        assert oracle.trees_from_result(res0, n) == want
        # B = n -> roots only
        r1 = oracle.select_literal(co, cp, cf, rng.uniform(0, 9, n), 8, 9, n)
        assert r1["tree_offsets"].tolist() == list(range(n + 1))
        # B >= N -> everything
        r2 = oracle.select_literal(co, cp, cf, rng.uniform(0, 9, n), 8, 9, N + 5)
        assert int(r2["tree_offsets"][-1]) == N
    with pytest.raises(ValueError):
        oracle.select_literal(np.array([0, 1, 2], np.int32), [0, 0], [1, 1], [0, 0], 3, 3, 1)


def test_monotone_mass_in_budget():
    """total selected f-hat does not decrease as B grows."""
    rng = np.random.default_rng(9)
    for _ in range(60):
        n = int(rng.integers(1, 5))
        F = synth.random_forest(rng, n, 10)
        co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
        A = rng.uniform(0, 4, n)
        prev = -1.0
        for B in range(n, int(co[-1]) + 2):
            res = oracle.select_literal(co, cp, cf, A, 4, 3, B)
            mass = sum(float(cf[co[i] + j]) for i, s in enumerate(oracle.trees_from_result(res, n)) for j in s)
            assert mass >= prev - 1e-9
            prev = mass


def test_beam_forest_c3_sizes():
    """The c3 generator + literal select give a ragged 2..64 size mix under B=4096."""
    rng = synth.rng_for(2)
    F = synth.beam_forest(rng, 64, 8, 8, 1.0, 8.0, with_targets=False)
    A = synth.slo_mix(rng, 64)
    res = oracle.select_literal(F["cand_offsets"], F["cand_parent"], F["cand_prob"], A, 8, 63, 1024)
    K = np.diff(res["tree_offsets"])
    assert K.sum() <= 1024 and K.min() >= 1 and K.max() <= 65
    _check_invariants(F["cand_offsets"], F["cand_parent"], F["cand_prob"], A, 8, 63, 1024, res)


# --------------------------------------------------------------------------- NEXT-4 variants (R24)
def _lexsort_topk_sets(F, caps):
    """Independent reference: per request, np.lexsort by (-f, index) over the
    non-root candidates, first caps[i] -- no loop of the oracle's."""
    co, cf = F["cand_offsets"], F["cand_prob"]
    out = []
    for i in range(len(co) - 1):
        idx = np.arange(1, co[i + 1] - co[i])
        f = cf[co[i] + idx].astype(np.float64)
        order = idx[np.lexsort((idx, -f))]
        out.append({0} | set(order[: max(0, int(caps[i]))].tolist()))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_per_request_greedy_is_lexsort_topk(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 30))
    F = synth.random_forest(rng, n, int(rng.integers(2, 40)), tie_prob=float(rng.choice([0.0, 0.6])))
    caps = rng.integers(0, 45, n)
    res = oracle.select_per_request_greedy(F["cand_offsets"], F["cand_parent"], F["cand_prob"], caps)
    got = oracle.trees_from_result(res, n)
    assert got == _lexsort_topk_sets(F, caps)
    # ancestor-closed, topological emission, compact parents point backwards
    to = res["tree_offsets"]
    for i in range(n):
        seg = slice(to[i], to[i + 1])
        assert (res["tree_parent"][seg][1:] < np.arange(1, to[i + 1] - to[i])).all()
        assert (np.diff(res["tree_src"][seg]) > 0).all()
    np.testing.assert_array_equal(res["kept"], np.diff(to) - 1)


def test_equal_greedy_caps_and_single_request_identity():
    """EqualGreedy splits B evenly (sum of shares = B); with one request it is
    GlobalGreedy (every A <= 1: Alg. 2's SLO stage is inert, P-sel-4)."""
    for n, B in ((7, 30), (3, 3), (5, 64), (1, 9)):
        caps = oracle.equal_greedy_caps(n, B)
        assert int((caps + 1).sum()) == B and caps.max() - caps.min() <= 1
    rng = np.random.default_rng(77)
    for _ in range(20):
        F = synth.random_forest(rng, 1, 30, tie_prob=0.3)
        N = int(F["cand_offsets"][-1])
        B = int(rng.integers(1, N + 3))
        eg = oracle.select_per_request_greedy(F["cand_offsets"], F["cand_parent"], F["cand_prob"],
                                              oracle.equal_greedy_caps(1, B))
        gg = oracle.select_literal(F["cand_offsets"], F["cand_parent"], F["cand_prob"], [0.5], 3, 0, B)
        np.testing.assert_array_equal(eg["tree_src"], gg["tree_src"])
        np.testing.assert_array_equal(eg["tree_parent"], gg["tree_parent"])
    with pytest.raises(ValueError):
        oracle.equal_greedy_caps(4, 3)
