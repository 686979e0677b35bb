"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs.  Select and accept are bit-exact; attention
max-abs error <= 2e-2 (bf16 inputs) or <= 1e-5 (fp32), per BASELINE north_star.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.helpers import bf16_bits, dev, oracle_attn, workload_to_device

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
F32_TOL = 1e-5


@pytest.fixture(scope="module")
def ada():
    import paper_2501_12162_b200 as ada
    ada.lib()
    return ada


# --------------------------------------------------------------------------- tcgen05 building blocks
@pytest.mark.parametrize("n,k,mn", [(64, 128, 0), (128, 128, 0), (64, 64, 0), (128, 64, 1), (64, 64, 1),
                                    (128, 128, 1), (128, 128, 3), (64, 64, 3), (128, 64, 2),
                                    (64, 128, 4), (128, 128, 4), (64, 64, 4), (128, 128, 5), (128, 64, 5),
                                    (128, 128, 7), (128, 64, 7), (64, 128, 6)])
def test_umma_selftest(ada, n, k, mn):
    """bit 0: B MN-major (the PV/V form); bit 1: A staged in TMEM (the P form);
    bit 2: the CTA pair (tcgen05.mma.cta_group::2, M = 256, B split along N)."""
    g = torch.Generator(device="cpu").manual_seed(n * 7 + k + mn)
    a = torch.randn(256 if mn & 4 else 128, k, generator=g).to(torch.bfloat16)
    b = torch.randn((k, n) if mn & 1 else (n, k), generator=g).to(torch.bfloat16)
    d = ada.selftest_umma(a.cuda(), b.cuda(), n, k, mn).cpu()
    ref = a.double() @ (b.double() if mn & 1 else b.double().T)
    torch.cuda.synchronize()
    assert torch.allclose(d.double(), ref, atol=1e-3, rtol=1e-4), (d - ref).abs().max()


# --------------------------------------------------------------------------- speculation (beam)
def _rand_probs(rng, shape, sigma, ties):
    z = rng.normal(0.0, sigma, shape)
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    p = e / e.sum(axis=-1, keepdims=True)
    if ties:  # quantise: many exactly equal probabilities (and zeros) -> key ties resolved by index
        p = np.floor(p * 64.0) / 64.0
    return p.astype(np.float32)


@pytest.mark.parametrize("V,width,n,d,ties", [(1000, 8, 6, 4, False), (1000, 8, 5, 3, True),
                                              (8195, 2, 3, 3, False), (20, 16, 4, 3, False),
                                              (5, 1, 3, 4, True), (128256, 8, 3, 2, False),
                                              # > 4 CTAs per SM of rows (layer 2: 640 / 608 rows): the LDGSTS-ring scan
                                              (3000, 8, 80, 3, False), (4096, 8, 76, 2, True)])
def test_beam_layers_bit_exact(ada, V, width, n, d, ties):
    """d speculation layers on the GPU (as_beam_step) == the oracle's beam step
    applied layer by layer: parents, tokens and f-hat bit-exact."""
    rng = np.random.default_rng(V + width + d)
    stride = 1 + d * width
    par = np.zeros(n * stride, np.int32)
    prob = np.zeros(n * stride, np.float32)
    tok = np.zeros(n * stride, np.int32)
    prob[::stride] = 1.0
    tok[::stride] = rng.integers(0, V, n)
    g_par, g_prob, g_tok = dev(par), dev(prob), dev(tok)
    ws = None
    for layer in range(1, d + 1):
        w_in = 1 if layer == 1 else width
        P = _rand_probs(rng, (n, w_in, V), float(rng.uniform(0.5, 4.0)), ties)
        ws = ada.beam_step(layer, width, dev(P), g_par, g_prob, g_tok, stride, workspace=ws)
        base_prev = 0 if layer == 1 else 1 + (layer - 2) * width
        base_new = 1 + (layer - 1) * width
        for i in range(n):
            fpar = prob[i * stride + base_prev: i * stride + base_prev + w_in]
            pr, tk, fv = oracle.beam_step(P[i], fpar, width)
            k = len(pr)
            o = i * stride + base_new
            par[o:o + k] = base_prev + pr
            tok[o:o + k] = tk
            prob[o:o + k] = fv
    assert ada.check_device_error(ws)[0] == 0
    np.testing.assert_array_equal(g_par.cpu().numpy(), par)
    np.testing.assert_array_equal(g_tok.cpu().numpy(), tok)
    np.testing.assert_array_equal(g_prob.cpu().numpy().view(np.int32), prob.view(np.int32))


def test_beam_then_select(ada):
    """Speculation feeds selection: the GPU-built forest selected on the GPU ==
    the oracle's select on the oracle-built forest."""
    rng = np.random.default_rng(5)
    n, d, width, V = 16, 5, 4, 3000
    stride = 1 + d * width
    prob = np.zeros(n * stride, np.float32)
    prob[::stride] = 1.0
    g_par, g_prob = dev(np.zeros(n * stride, np.int32)), dev(prob)
    g_tok = dev(np.zeros(n * stride, np.int32))
    for layer in range(1, d + 1):
        P = _rand_probs(rng, (n, 1 if layer == 1 else width, V), 2.0, False)
        ada.beam_step(layer, width, dev(P), g_par, g_prob, g_tok, stride)
    F = dict(cand_offsets=np.arange(0, (n + 1) * stride, stride, dtype=np.int32),
             cand_parent=g_par.cpu().numpy(), cand_prob=g_prob.cpu().numpy())
    A = rng.uniform(0.5, 3.0, n)
    got = _gpu_select(ada, F, A, d, 10, n * 8)
    _assert_select_equal(F, A, d, 10, n * 8, got)


# --------------------------------------------------------------------------- select
def _gpu_select(ada, F, A, d, n_max, B):
    co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
    tok = F.get("cand_token")
    out = ada.select_trees(dev(co), dev(cp), dev(cf), dev(np.asarray(A, np.float64)), d, n_max, B,
                           cand_token=None if tok is None else dev(tok))
    code, req = ada.check_device_error(out["workspace"])
    assert code == 0, (code, req)
    return {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}


def _assert_select_equal(F, A, d, n_max, B, got):
    ref = oracle.select_literal(F["cand_offsets"], F["cand_parent"], F["cand_prob"], A, d, n_max, B)
    n = len(F["cand_offsets"]) - 1
    used = int(ref["tree_offsets"][-1])
    np.testing.assert_array_equal(got["tree_offsets"][: n + 1], ref["tree_offsets"])
    np.testing.assert_array_equal(got["tree_src"][:used], ref["tree_src"])
    np.testing.assert_array_equal(got["tree_parent"][:used], ref["tree_parent"])
    np.testing.assert_array_equal(got["tree_depth"][:used], ref["tree_depth"])
    np.testing.assert_array_equal(got["slo_count"][:n], ref["slo_count"])
    if F.get("cand_token") is not None:
        to = ref["tree_offsets"]
        req = np.repeat(np.arange(n), np.diff(to))
        want = F["cand_token"][F["cand_offsets"][req] + ref["tree_src"]]
        np.testing.assert_array_equal(got["tree_token"][:used], want)
    return ref


def test_select_fig4(ada):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig4.json")))
    offs = [0]
    par, prob = [], []
    for r in g["requests"]:
        par += r["parent"]
        prob += r["prob"]
        offs.append(offs[-1] + len(r["parent"]))
    F = dict(cand_offsets=np.array(offs, np.int32), cand_parent=np.array(par, np.int32),
             cand_prob=np.array(prob, np.float32))
    got = _gpu_select(ada, F, g["slo_deficit"], g["depth_d"], g["n_max"], g["budget"])
    ref = _assert_select_equal(F, g["slo_deficit"], g["depth_d"], g["n_max"], g["budget"], got)
    assert got["slo_count"][:2].tolist() == g["expected"]["slo_count"]
    assert int(ref["tree_offsets"][-1]) == g["expected"]["used"]


@pytest.mark.parametrize("cfg", ["c1", "c1slo", "c2", "c3", "c4", "c5"])
def test_select_configs(ada, cfg):
    rng = synth.rng_for(["c1", "c1slo", "c2", "c3", "c4", "c5"].index(cfg), salt=3)
    if cfg.startswith("c1"):
        F = synth.beam_forest(rng, 1, 3, 3)
        A, n_max, B, d = ([0.5], 7, 8, 3) if cfg == "c1" else ([2.5], 7, 8, 3)
    elif cfg == "c2":
        F = synth.beam_forest(rng, 64, 8, 8, 1.0, 4.0)
        A, n_max, B, d = np.full(64, 9.0), 31, 2048, 8
    elif cfg == "c3":
        F = synth.beam_forest(rng, 256, 8, 8, 1.0, 8.0)
        A, n_max, B, d = synth.slo_mix(rng, 256), 63, 4096, 8
    elif cfg == "c4":
        F = synth.beam_forest(rng, 128, 8, 8, 1.0, 4.0)
        A, n_max, B, d = np.full(128, 9.0), 63, 8192, 8
    else:
        F = synth.beam_forest(rng, 32, 8, 8, 1.0, 4.0)
        A, n_max, B, d = np.full(32, 9.0), 63, 2048, 8
    got = _gpu_select(ada, F, A, d, n_max, B)
    ref = _assert_select_equal(F, A, d, n_max, B, got)
    if cfg == "c2":
        assert (np.diff(ref["tree_offsets"]) == 32).all()


@pytest.mark.parametrize("seed", range(6))
def test_select_fuzz(ada, seed):
    rng = np.random.default_rng(100 + seed)
    for it in range(40):
        n = int(rng.integers(1, [8, 40, 300, 1200, 64, 2][seed]))
        maxn = int([12, 40, 80, 6, 257, 257][seed])
        F = synth.random_forest(rng, n, maxn, tie_prob=float(rng.choice([0.0, 0.5])))
        N = int(F["cand_offsets"][-1])
        F["cand_token"] = rng.integers(0, 128256, N).astype(np.int32)
        A = rng.uniform(-1, 7, n)
        if rng.random() < 0.5:
            A[rng.integers(0, n, max(1, n // 3))] = A[0]
        d = int(rng.integers(1, 9))
        n_max = int(rng.integers(0, 70))
        B = int(rng.integers(n, N + 5))
        got = _gpu_select(ada, F, A, d, n_max, B)
        _assert_select_equal(F, A, d, n_max, B, got)


@pytest.mark.parametrize("seed", range(4))
def test_select_radix_shared_key_bits(ada, seed):
    """The throughput stage's radix select starts below the key bits all tails
    share (AND / OR over the cluster): f-hat squeezed into [0.5, 0.5 + 2^-s] by a
    monotone map (parent >= child and exact ties preserved) leaves only the low
    mantissa bits and the request/index word to decide -- bit-exact vs Alg. 2."""
    rng = np.random.default_rng(900 + seed)
    for it in range(12):
        n = int(rng.integers(2, [40, 300, 700, 2][seed] + 1))
        F = synth.random_forest(rng, n, int(rng.integers(8, 80)), tie_prob=float(rng.choice([0.0, 0.5])))
        sq = [4, 10, 18, 23][int(rng.integers(0, 4))]
        F["cand_prob"] = (np.float32(0.5) + F["cand_prob"] * np.float32(2.0 ** -sq)).astype(np.float32)
        N = int(F["cand_offsets"][-1])
        A = rng.uniform(-1, 3, n)
        d = int(rng.integers(1, 9))
        n_max = int(rng.integers(0, 20))
        B = int(rng.integers(n, N + 5))
        got = _gpu_select(ada, F, A, d, n_max, B)
        _assert_select_equal(F, A, d, n_max, B, got)


@pytest.mark.parametrize("seed", range(4))
def test_select_global_greedy_is_lexsort_topk(ada, seed):
    """NEXT-4 GlobalGreedy through select_global_greedy: every root,
    then the global top-(B - n) non-root candidates by (f-hat desc, request asc,
    index asc) -- computed here with np.lexsort, not by the oracle's Alg. 2.
    The set is ancestor-closed because f-hat never grows down a path and a
    parent's index precedes its child's (P-sel-4, R8)."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(1, [5, 60, 400, 2000][seed]))
    F = synth.random_forest(rng, n, [20, 60, 120, 9][seed], tie_prob=[0.0, 0.5, 0.2, 0.7][seed])
    co, cp, cf = F["cand_offsets"], F["cand_parent"], F["cand_prob"]
    N = int(co[-1])
    B = n + int(rng.integers(0, N - n + 1))
    out = ada.select_global_greedy(dev(co), dev(cp), dev(cf), B)
    assert ada.check_device_error(out["workspace"])[0] == 0
    req = np.repeat(np.arange(n), np.diff(co))
    loc = np.arange(N) - co[req]
    nonroot = np.nonzero(loc > 0)[0]
    order = nonroot[np.lexsort((loc[nonroot], req[nonroot], -cf[nonroot].astype(np.float64)))]
    chosen = np.zeros(N, bool)
    chosen[co[:-1]] = True
    chosen[order[:B - n]] = True
    to = out["tree_offsets"].cpu().numpy()
    src = out["tree_src"].cpu().numpy()
    np.testing.assert_array_equal(np.diff(to), np.bincount(req[chosen], minlength=n))
    for i in range(n):
        np.testing.assert_array_equal(src[to[i]:to[i + 1]], loc[chosen & (req == i)])
    np.testing.assert_array_equal(out["slo_count"].cpu().numpy()[:n], 0)


@pytest.mark.parametrize("seed", range(5))
def test_select_topm_and_equal_greedy_bit_exact(ada, seed):
    """NEXT-4 variants (reading R24) through as_select_topm: Eagle-2 top-m and
    EqualGreedy(B) == the oracle's per-request GetTop loop, bit for bit (src,
    compact parents, depth, tokens, kept), incl. exact f-hat ties, caps larger
    than the candidate count, and a batch past the shared staging area."""
    rng = np.random.default_rng(1300 + seed)
    n, maxn = [(5, 20), (60, 70), (300, 66), (2500, 100), (1, 257)][seed]
    F = synth.random_forest(rng, n, maxn, tie_prob=0.4, min_nodes=1)
    N = int(F["cand_offsets"][-1])
    tok = rng.integers(0, 128256, N).astype(np.int32)
    co, cp, cf = dev(F["cand_offsets"]), dev(F["cand_parent"]), dev(F["cand_prob"])
    for mode in ("topm", "equal"):
        if mode == "topm":
            m = int(rng.integers(0, maxn + 3))
            caps = np.full(n, m)
            out = ada.select_topm(co, cp, cf, m, cand_token=dev(tok))
        else:
            B = n + int(rng.integers(0, max(1, N - n + 1)))
            caps = oracle.equal_greedy_caps(n, B)
            out = ada.select_equal_greedy(co, cp, cf, B, cand_token=dev(tok))
        assert ada.check_device_error(out["workspace"])[0] == 0
        ref = oracle.select_per_request_greedy(F["cand_offsets"], F["cand_parent"], F["cand_prob"], caps)
        used = int(ref["tree_offsets"][-1])
        np.testing.assert_array_equal(out["tree_offsets"].cpu().numpy(), ref["tree_offsets"])
        np.testing.assert_array_equal(out["tree_src"].cpu().numpy()[:used], ref["tree_src"])
        np.testing.assert_array_equal(out["tree_parent"].cpu().numpy()[:used], ref["tree_parent"])
        np.testing.assert_array_equal(out["tree_depth"].cpu().numpy()[:used], ref["tree_depth"])
        np.testing.assert_array_equal(out["kept"].cpu().numpy()[:n], ref["kept"])
        req = np.repeat(np.arange(n), np.diff(ref["tree_offsets"]))
        np.testing.assert_array_equal(out["tree_token"].cpu().numpy()[:used],
                                      tok[F["cand_offsets"][req] + ref["tree_src"]])


def test_select_exact_sum_guards(ada):
    """Both desired_i paths of the kernel: the warp fp64 scan is used only when
    every f-hat >= 2^-24 and 1 + sum < 64 (R9); chains of f-hat = 1.0 (sums past
    64) and tiny f-hat (< 2^-24) must take the sequential loop and still match."""
    rng = np.random.default_rng(7)
    # (a) chains with f = 1.0 everywhere: n_acc reaches 1 + 200 > 64
    n, K = 5, 201
    F = dict(cand_offsets=np.arange(0, (n + 1) * K, K, dtype=np.int32),
             cand_parent=np.concatenate([[0] + list(range(K - 1))] * n).astype(np.int32),
             cand_prob=np.ones(n * K, np.float32))
    for A, d, n_max in ((150.0, 300, 250), (70.5, 300, 250), (30.0, 300, 250), (300.0, 100, 90)):
        got = _gpu_select(ada, F, np.full(n, A), d, n_max, n * K)
        _assert_select_equal(F, np.full(n, A), d, n_max, n * K, got)
    # (b) tiny path probabilities (< 2^-24) mixed with large ones
    for it in range(10):
        F = synth.random_forest(rng, 40, 60)
        f = F["cand_prob"].copy()
        co = F["cand_offsets"]
        for i in range(40):
            if rng.random() < 0.5:
                # scale a whole request's non-root f by 2^-30 (keeps f(child) <= f(parent))
                f[co[i] + 1: co[i + 1]] = (f[co[i] + 1: co[i + 1]].astype(np.float64) * 2.0 ** -30).astype(np.float32)
        F["cand_prob"] = f
        A = rng.uniform(0.5, 4.0, 40)
        n_max = int(rng.integers(1, 60))
        B = int(rng.integers(40, 1500))
        got = _gpu_select(ada, F, A, 8, n_max, B)
        _assert_select_equal(F, A, 8, n_max, B, got)
    # (c) the SLO threshold inside a tail of tiny f-hat: chains 0.5, 0.25, 0.125, then
    # 40 entries of 2^-26 (decreasing by ulps); A puts the crossing inside the tiny tail,
    # exactly on a partial sum, or just out of reach (the kernel's bound must not cut it)
    K = 44
    big = [0.5, 0.25, 0.125]
    tiny = [np.float32(2.0 ** -26) * np.float32(1 - 2.0 ** -20 * j) for j in range(K - 4)]
    chain = np.array([1.0] + big + tiny, np.float32)
    run = 1.0 + sum(big)
    As = [run + 1.5 * 2.0 ** -26, run + 7 * 2.0 ** -26, run + float(np.sum(np.array(tiny[:20], np.float64))),
          run + 39.9 * 2.0 ** -26, run + 40.5 * 2.0 ** -26, run + 2.0 ** -30, run - 2.0 ** -40, run + 1e-3]
    n = len(As)
    F = dict(cand_offsets=np.arange(0, (n + 1) * K, K, dtype=np.int32),
             cand_parent=np.concatenate([[0] + list(range(K - 1))] * n).astype(np.int32),
             cand_prob=np.tile(chain, n))
    got = _gpu_select(ada, F, np.array(As), 100, 60, n * K)
    _assert_select_equal(F, np.array(As), 100, 60, n * K, got)


@pytest.mark.parametrize("n,maxn", [(4096, 5), (2500, 100)])
def test_select_large_batches(ada, n, maxn):
    """Cluster of 16 CTAs with several requests per warp (4096 x 5), and a batch
    whose candidates overflow the per-CTA shared staging area (2500 x ~100):
    the kernel then keeps pi_i in the workspace -- same results."""
    rng = np.random.default_rng(n)
    F = synth.random_forest(rng, n, maxn, tie_prob=0.3, min_nodes=max(1, maxn - 10))
    A = rng.uniform(-1, 5, n)
    N = int(F["cand_offsets"][-1])
    for n_max, B in ((3, n + min(3000, (N - n) // 3)), (40, n + 1500)):
        got = _gpu_select(ada, F, A, 8, n_max, B)
        _assert_select_equal(F, A, 8, n_max, B, got)


# --------------------------------------------------------------------------- accept
def _accept_inputs(rng, n, maxK, vocab=50, dtype=np.float32, n_kv=2, d=64, ps=16, L_max=70):
    sizes = rng.integers(1, maxK + 1, n)
    to = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    R = int(to[-1])
    par = np.concatenate([synth.random_tree_parents(rng, int(k), shape=rng.choice(["random", "chain", "star"]))
                          for k in sizes]).astype(np.int32)
    toks = np.zeros(R, np.int32)
    for i in range(n):
        for p in range(int(sizes[i])):
            kids = [c for c in range(1, int(sizes[i])) if par[to[i] + c] == p]
            vals = rng.permutation(vocab)[: len(kids)]
            if rng.random() < 0.2 and len(kids) > 1:
                vals[1] = vals[0]  # duplicate sibling token: lowest index must win
            for c, v in zip(kids, vals):
                toks[to[i] + c] = v
    tgt = rng.integers(0, vocab, R).astype(np.int32)
    for i in range(n):  # make walks go deep: 75% of nodes target one of their children
        for p in range(int(sizes[i])):
            kids = [c for c in range(1, int(sizes[i])) if par[to[i] + c] == p]
            if kids and rng.random() < 0.75:
                tgt[to[i] + p] = toks[to[i] + kids[int(rng.integers(0, len(kids)))]]
    kv_len = rng.integers(0, L_max, n).astype(np.int32)
    table, n_pages = synth.paged_kv(rng, kv_len, ps, extra_slots=maxK + 2)
    shape_t, shape_c = (R, n_kv, d), (n_pages, n_kv, ps, d)
    if dtype == np.float32:
        kt, vt = rng.standard_normal(shape_t).astype(np.float32), rng.standard_normal(shape_t).astype(np.float32)
        kc, vc = rng.standard_normal(shape_c).astype(np.float32), rng.standard_normal(shape_c).astype(np.float32)
    else:
        kt = synth.bf16_round(rng.standard_normal(shape_t).astype(np.float32))
        vt = synth.bf16_round(rng.standard_normal(shape_t).astype(np.float32))
        kc = synth.bf16_round(rng.standard_normal(shape_c).astype(np.float32))
        vc = synth.bf16_round(rng.standard_normal(shape_c).astype(np.float32))
    return dict(to=to, par=par, toks=toks, tgt=tgt, kv_len=kv_len, table=table, kt=kt, vt=vt, kc=kc, vc=vc)


@pytest.mark.parametrize("kv_dtype", [torch.float32, torch.bfloat16])
def test_accept_fused_tokens(ada, kv_dtype):
    rng = np.random.default_rng(11)
    for it in range(6):
        n = int(rng.integers(1, 200))
        X = _accept_inputs(rng, n, int(rng.integers(1, 65)), dtype=np.float32 if kv_dtype == torch.float32 else "bf16")
        max_path = 64
        ref = oracle.accept_walk(X["to"], X["par"], X["toks"], target_tokens=X["tgt"], max_path=max_path)
        kc_g, vc_g, kl_g = dev(X["kc"], kv_dtype), dev(X["vc"], kv_dtype), dev(X["kv_len"])
        res = ada.accept_tokens(ada.AS_ACCEPT_FUSED, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                                target_tokens=dev(X["tgt"]), max_path=max_path, k_tree=dev(X["kt"], kv_dtype),
                                v_tree=dev(X["vt"], kv_dtype), k_cache=kc_g, v_cache=vc_g, page_table=dev(X["table"]),
                                kv_len=kl_g)
        assert ada.check_device_error(res["workspace"])[0] == 0
        np.testing.assert_array_equal(res["accept_len"].cpu().numpy()[:n], ref["accept_len"])
        np.testing.assert_array_equal(res["accept_path"].cpu().numpy()[:n], ref["accept_path"])
        np.testing.assert_array_equal(res["bonus_token"].cpu().numpy()[:n], ref["bonus_token"])
        # commit, byte-exact (oracle on the same byte patterns)
        if kv_dtype == torch.bfloat16:
            to_bits = lambda a: bf16_bits(torch.from_numpy(a).to(torch.bfloat16))
            kc, vc, kt, vt = (to_bits(X[k]) for k in ("kc", "vc", "kt", "vt"))
            got_k, got_v = bf16_bits(kc_g), bf16_bits(vc_g)
        else:
            kc, vc, kt, vt = (X[k].copy() for k in ("kc", "vc", "kt", "vt"))
            got_k, got_v = kc_g.cpu().numpy(), vc_g.cpu().numpy()
        kl = X["kv_len"].copy()
        assert oracle.commit(X["to"], ref["accept_len"], ref["accept_path"], kt, vt, kc, vc, X["table"], kl) == 0
        np.testing.assert_array_equal(kl_g.cpu().numpy(), kl)
        np.testing.assert_array_equal(got_k.view(np.uint8), kc.view(np.uint8))
        np.testing.assert_array_equal(got_v.view(np.uint8), vc.view(np.uint8))


@pytest.mark.parametrize("ldt", [torch.float32, torch.bfloat16])
def test_accept_logits_greedy(ada, ldt):
    rng = np.random.default_rng(12)
    n = 37
    X = _accept_inputs(rng, n, 20, vocab=3000)
    R = int(X["to"][-1])
    vocab = 3001  # odd: exercises the unaligned tail path
    logits = rng.standard_normal((R, vocab)).astype(np.float32)
    logits[np.arange(R), X["tgt"]] = 9.0
    tie = rng.random(R) < 0.3  # exact ties: the lower index must win
    alt = rng.integers(0, vocab, R)
    logits[tie, alt[tie]] = 9.0
    if ldt == torch.bfloat16:
        logits = synth.bf16_round(logits)
    ref = oracle.accept_walk(X["to"], X["par"], X["toks"], target_logits=logits, max_path=32)
    res = ada.accept_tokens(ada.AS_ACCEPT_WALK_ONLY, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                            target_logits=dev(logits, ldt), max_path=32)
    assert ada.check_device_error(res["workspace"])[0] == 0
    np.testing.assert_array_equal(res["accept_len"].cpu().numpy()[:n], ref["accept_len"])
    np.testing.assert_array_equal(res["accept_path"].cpu().numpy()[:n], ref["accept_path"])
    np.testing.assert_array_equal(res["bonus_token"].cpu().numpy()[:n], ref["bonus_token"])


def test_accept_sharded_walk_then_commit_equals_fused(ada):
    """WALK_ONLY over request shards + COMMIT_ONLY over all == FUSED (the
    multi-GPU protocol with the all-gather replaced by local copies)."""
    rng = np.random.default_rng(13)
    n = 50
    X = _accept_inputs(rng, n, 30, dtype="bf16")
    args = dict(k_tree=dev(X["kt"], torch.bfloat16), v_tree=dev(X["vt"], torch.bfloat16),
                page_table=dev(X["table"]))
    kc1, vc1, kl1 = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16), dev(X["kv_len"])
    fused = ada.accept_tokens(ada.AS_ACCEPT_FUSED, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                              target_tokens=dev(X["tgt"]), max_path=24, k_cache=kc1, v_cache=vc1, kv_len=kl1, **args)
    al = torch.full((n,), -5, dtype=torch.int32, device="cuda")
    ap = torch.full((n, 24), -5, dtype=torch.int32, device="cuda")
    bt = torch.full((n,), -5, dtype=torch.int32, device="cuda")
    for b, e in [(0, 17), (17, 34), (34, 50)]:
        ada.accept_tokens(ada.AS_ACCEPT_WALK_ONLY, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                          target_tokens=dev(X["tgt"]), max_path=24, req_range=(b, e), accept_len=al,
                          accept_path=ap, bonus_token=bt)
    kc2, vc2, kl2 = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16), dev(X["kv_len"])
    ada.accept_tokens(ada.AS_ACCEPT_COMMIT_ONLY, dev(X["to"]), max_path=24, accept_len=al, accept_path=ap,
                      k_cache=kc2, v_cache=vc2, kv_len=kl2, n_tree_rows=int(X["to"][-1]), **args)
    assert torch.equal(al, fused["accept_len"]) and torch.equal(ap, fused["accept_path"])
    assert torch.equal(bt, fused["bonus_token"])
    assert torch.equal(kl1, kl2) and torch.equal(kc1, kc2) and torch.equal(vc1, vc2)
    # the record form used across GPUs: shards walk into their rows of one
    # [world*s, 2 + max_path] buffer (the all-gather is the identity on one GPU),
    # then every request is committed from the records; kv_len_out out of place
    world, s = 3, 17
    rec = torch.full((world * s, 26), -7, dtype=torch.int32, device="cuda")
    for r in range(world):
        b, e = min(n, r * s), min(n, r * s + s)
        ada.accept_tokens(ada.AS_ACCEPT_WALK_RECORDS, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                          target_tokens=dev(X["tgt"]), max_path=24, req_range=(b, e), accept_path=rec)
    assert torch.equal(rec[:n, 0], fused["accept_len"]) and torch.equal(rec[:n, 1], fused["bonus_token"])
    assert torch.equal(rec[:n, 2:], fused["accept_path"])
    kc3, vc3, kl3 = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16), dev(X["kv_len"])
    kl3_out = torch.full_like(kl3, -1)
    ada.accept_tokens(ada.AS_ACCEPT_COMMIT_RECORDS, dev(X["to"]), max_path=24, accept_path=rec, k_cache=kc3,
                      v_cache=vc3, kv_len=kl3, kv_len_out=kl3_out, n_tree_rows=int(X["to"][-1]), **args)
    assert torch.equal(kl3, dev(X["kv_len"]))  # input untouched
    assert torch.equal(kl3_out, kl1) and torch.equal(kc3, kc1) and torch.equal(vc3, vc1)


# --------------------------------------------------------------------------- attention
ATTN_CASES = [
    # (sizes, kv_lens, n_q, n_kv, d, page_size, shape, q_scale)
    ([8], [128], 4, 4, 64, 16, "random", 1.0),                     # BASELINE config 1
    ([8], [128], 4, 2, 64, 16, "random", 1.0),                     # c1 GQA variant
    ([1, 1, 2], [0, 1, 63], 4, 4, 64, 16, "random", 1.0),          # L=0, root-only
    ([5, 17, 33], [64, 65, 127], 8, 2, 128, 32, "chain", 1.0),     # tile boundaries, chains
    ([40, 7], [300, 129], 8, 1, 128, 128, "star", 1.0),            # G=8, star, page 128
    ([64, 3, 128], [200, 5, 77], 4, 1, 128, 64, "random", 4.0),    # multi m-tile, K=128, peaky
    ([128], [96], 16, 1, 128, 16, "chain", 1.0),                   # G=16, 16 m-tiles, deep chain
    ([9, 31, 2, 64, 15], [1000, 33, 0, 511, 2049], 32, 8, 128, 64, "random", 1.0),  # Llama-3-8B heads
    # NEXT-4: trees past 128 nodes (3-4 tree tiles, up to 8 q-tiles per head)
    ([256, 129, 192, 3], [300, 64, 0, 1000], 8, 2, 128, 64, "random", 1.0),
    ([255, 200], [130, 17], 4, 4, 64, 32, "chain", 2.0),           # deep chains, d=64
    ([257 - 1, 130], [64, 700], 32, 8, 128, 64, "star", 1.0),       # 8B heads, G=4: 8 q-tiles
]


def _attn_case(case, bf16, seed):
    sizes, kv_lens, n_q, n_kv, d, ps, shape, qs = case
    rng = np.random.default_rng(seed)
    return synth.tree_workload(rng, sizes, kv_lens, n_q, n_kv, d, ps, shape=shape, bf16=bf16, q_scale=qs)


@pytest.mark.parametrize("ci", range(len(ATTN_CASES)))
def test_attn_fp32(ada, ci):
    w = _attn_case(ATTN_CASES[ci], False, 300 + ci)
    scale = np.float32(1.0 / np.sqrt(w["q"].shape[2]))
    ref, ref_lse = oracle_attn(w, scale)
    g = workload_to_device(w, torch.float32)
    ws = ada.Workspace(256)
    out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                    g["kv_len"], g["tree_offsets"], g["tree_parent"], scale, want_lse=True,
                                    workspace=ws)
    assert ada.check_device_error(ws)[0] == 0
    err = np.abs(out.cpu().numpy() - ref).max()
    assert err <= F32_TOL, err
    assert np.abs(lse.cpu().numpy() - ref_lse).max() <= 1e-4


def _sched(shape, split=None):
    """as_tree_verify_attn_sched overrides: "1"/"2" = q-tiles per CTA, "cs2"/"cs4" =
    clusters of one-q-tile CTAs sharing K/V by multicast; split "0" = whole units."""
    parts = []
    if shape == "2cs2":  # two NQ=2 CTAs of a cluster: four q-tiles share each K/V fetch
        parts.append("nq=2,cs=2")
    elif shape.startswith("cs"):
        parts.append(f"cs={shape[2:]}")
    elif shape != "auto":
        parts.append(f"nq={shape}")
    if split is not None:
        parts.append(f"split={0 if split == '0' else 1}")
    return ",".join(parts) or None


@pytest.mark.parametrize("ci", range(1, len(ATTN_CASES)))
@pytest.mark.parametrize("nq", ["auto", "1", "2", "cs2", "cs4", "2cs2"])
def test_attn_bf16(ada, ci, nq):
    """Every CTA shape: one q-tile per CTA (NQ=1), paired q-tiles sharing every
    K/V tile (NQ=2; odd q-tile counts leave the second group idle), and clusters
    of 2 / 4 one-q-tile CTAs fetching each K/V tile once and multicasting it
    (CTAs past a head's last q-tile only stream and release)."""
    sched = _sched(nq)
    w = _attn_case(ATTN_CASES[ci], True, 400 + ci)
    scale = np.float32(1.0 / np.sqrt(w["q"].shape[2]))
    ref, ref_lse = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                    g["kv_len"], g["tree_offsets"], g["tree_parent"], scale, want_lse=True,
                                    workspace=ws, schedule=sched)
    assert ada.check_device_error(ws)[0] == 0
    err = np.abs(out.float().cpu().numpy() - ref).max()
    assert err <= BF16_TOL, err
    assert np.abs(lse.cpu().numpy() - ref_lse).max() <= BF16_TOL


@pytest.mark.parametrize("nq,q_scale", [("auto", 4.0), ("auto", 8.0), ("1", 4.0), ("2", 4.0), ("2cs2", 4.0)])
def test_attn_bf16_long_context_peaky(ada, nq, q_scale):
    """c5-length prefixes (32k and 20k keys plus a short one) with peaky queries
    (q scaled 4x / 8x: a few keys dominate each row, so bf16 rounding of P and
    the lazy rescale matter most), Llama-3-8B heads, 64-node trees: every CTA
    shape against the fp64 oracle within the 2e-2 bound."""
    rng = np.random.default_rng(77 if q_scale == 4.0 else 78)
    w = synth.tree_workload(rng, [64, 33, 8], [32768, 20000, 4097], 32, 8, 128, 64, shape="random", bf16=True,
                            q_scale=q_scale)
    scale = np.float32(1.0 / np.sqrt(128))
    ref, ref_lse = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                    g["kv_len"], g["tree_offsets"], g["tree_parent"], scale, want_lse=True,
                                    workspace=ws, schedule=_sched(nq))
    assert ada.check_device_error(ws)[0] == 0
    err = np.abs(out.float().cpu().numpy() - ref).max()
    print(f"long-context peaky q_scale={q_scale} shape={nq}: max abs err {err:.5f} (bound {BF16_TOL})")
    assert err <= BF16_TOL, err
    assert np.abs(lse.cpu().numpy() - ref_lse).max() <= BF16_TOL


@pytest.mark.parametrize("nq", ["1", "2", "cs2", "2cs2"])
def test_attn_bf16_request_chunks(ada, nq):
    sched = _sched(nq)
    """More units than the kernel's per-CTA piece lists hold (n_kv * q-tiles *
    n_req > 64 * 2 * SMs): the library verifies the batch in request chunks;
    every request, including those at chunk edges, must match the oracle."""
    rng = np.random.default_rng(31)
    n = 700
    sizes = rng.integers(1, 6, n)
    sizes[::97] = 40  # a few multi-q-tile requests (G*K > 128)
    kv = rng.integers(0, 90, n)
    w = synth.tree_workload(rng, sizes, kv, 32, 8, 128, 64, bf16=True)
    scale = np.float32(1.0 / np.sqrt(128))
    ref, _ = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    out, _ = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                  g["kv_len"], g["tree_offsets"], g["tree_parent"], scale, workspace=ws, schedule=sched)
    assert ada.check_device_error(ws)[0] == 0
    assert np.abs(out.float().cpu().numpy() - ref).max() <= BF16_TOL


def test_attn_bf16_plan_capacity_chunks(ada):
    """More requests than one launch's schedule plan holds (head_dim 64, G = 1:
    few units per request, so the plan's per-request capacity binds before the
    per-CTA piece lists do): the library launches request chunks sized by both
    limits; every request matches the oracle and no device error is raised."""
    rng = np.random.default_rng(41)
    n = 2600
    sizes = rng.integers(1, 4, n)
    kv = rng.integers(0, 40, n)
    w = synth.tree_workload(rng, sizes, kv, 2, 2, 64, 16, bf16=True)
    scale = np.float32(1.0 / 8.0)
    ref, _ = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    out, _ = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                  g["kv_len"], g["tree_offsets"], g["tree_parent"], scale, workspace=ws)
    assert ada.check_device_error(ws)[0] == 0
    assert np.abs(out.float().cpu().numpy() - ref).max() <= BF16_TOL


@pytest.mark.parametrize("sk", ["0", "1", "2"])
@pytest.mark.parametrize("shape", ["1", "cs2", "2cs2"])
def test_attn_bf16_many_units(ada, sk, shape):
    """More units than CTAs (64 requests x 8 kv heads = 512 > 296 one-q-tile
    CTAs), ragged kv lengths, under every split setting (0: never
    split; 1/2: split-KV allowed -- not taken here, units outnumber CTAs), two
    launches on one workspace.  (A tail stream-K schedule for this regime was
    tried in commit 2530b31 and measured slower.)"""
    sched = _sched(shape, sk)
    rng = np.random.default_rng(57)
    n = 64
    sizes = rng.integers(20, 33, n)
    kv = rng.integers(500, 1200, n)
    kv[::9] = 0  # prefix-free requests among them
    w = synth.tree_workload(rng, sizes, kv, 32, 8, 128, 64, bf16=True)
    scale = np.float32(1.0 / np.sqrt(128))
    ref, ref_lse = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    for rep in range(2):  # the second launch reuses the (self-resetting) counters
        out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"],
                                        g["page_table"], g["kv_len"], g["tree_offsets"], g["tree_parent"], scale,
                                        want_lse=True, workspace=ws, schedule=sched)
        assert ada.check_device_error(ws)[0] == 0
        err = np.abs(out.float().cpu().numpy() - ref).max()
        assert err <= BF16_TOL, (rep, err)
        assert np.abs(lse.cpu().numpy() - ref_lse).max() <= 1e-2


def test_attn_bf16_deterministic_under_tail_pieces(ada):
    """c2's batch (512 one-q-tile units on 296 CTAs) runs the tail stream-K
    schedule, where the LAST piece of a cut unit to finish merges it: the merge
    combines the pieces in stream order whoever merges, so two launches (and a
    graph replay) give bit-identical outputs."""
    import bench
    W = bench.make_workload("c2", "cuda", seed_salt=3)
    bench.run_select(W)
    a = bench.run_attention(W).clone()
    for _ in range(3):
        W["ws_attn"] = ada.Workspace(W["ws_attn"].nbytes)
        b = bench.run_attention(W)
        torch.cuda.synchronize()
        used = int(W["sel"]["tree_offsets"][-1])
        assert torch.equal(a[:used], b[:used])


@pytest.mark.parametrize("ci", [4, 5, 8, 10])
@pytest.mark.parametrize("nq", ["1", "2"])
def test_attn_bf16_cta_pair(ada, ci, nq):
    """CTA pairs (as_attn_schedule.cta_pair): one tcgen05.mma.cta_group::2 (M = 256)
    per q-tile pair of a 2-CTA cluster, each CTA loading half of every K/V tile;
    1 or 2 q-tiles per CTA; odd q-tile counts leave the peer's half idle; trees
    up to 256 nodes, page sizes 64 / 128."""
    w = _attn_case(ATTN_CASES[ci], True, 900 + ci)
    scale = np.float32(1.0 / np.sqrt(w["q"].shape[2]))
    ref, ref_lse = oracle_attn(w, scale)
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    for rep in range(2):
        out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"],
                                        g["page_table"], g["kv_len"], g["tree_offsets"], g["tree_parent"], scale,
                                        want_lse=True, workspace=ws, schedule=f"pair=1,nq={nq}")
        assert ada.check_device_error(ws)[0] == 0
        err = np.abs(out.float().cpu().numpy() - ref).max()
        assert err <= BF16_TOL, (rep, err)
        assert np.abs(lse.cpu().numpy() - ref_lse).max() <= 1e-2


def test_attn_tree_too_big_is_flagged(ada):
    """K_i > AS_MAX_TREE (256): the request is skipped and AS_DEV_TREE_TOO_BIG
    reported with its index; the other requests are still verified."""
    w = _attn_case(([5, 257, 9], [40, 10, 70], 8, 2, 128, 64, "random", 1.0), True, 93)
    scale = np.float32(1.0 / np.sqrt(128))
    g = workload_to_device(w, torch.bfloat16)
    ws = ada.Workspace(256)
    out, _ = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                  g["kv_len"], g["tree_offsets"], g["tree_parent"], scale, workspace=ws)
    assert ada.check_device_error(ws) == (4, 1)
    to = w["tree_offsets"]
    keep = [0, 2]
    rows, ref, _ = oracle_attn(w, scale, requests=keep)
    got = out[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    assert np.abs(got - ref).max() <= BF16_TOL


def test_attn_bf16_nan_in_unused_cache_slots(ada):
    """Cache slots past kv_len may hold garbage (NaN): outputs must not see them."""
    w = _attn_case(([6, 9], [70, 33], 8, 2, 128, 64, "random", 1.0), True, 77)
    scale = np.float32(1.0 / np.sqrt(128))
    ref, _ = oracle_attn(w, scale)
    ps = 64
    for i, L in enumerate(w["kv_len"]):
        for t in range(int(L), w["page_table"].shape[1] * ps):
            pg = w["page_table"][i, t // ps]
            if pg >= 0:
                w["k_cache"][pg, :, t % ps] = np.nan
                w["v_cache"][pg, :, t % ps] = np.nan
    g = workload_to_device(w, torch.bfloat16)
    out, _ = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                  g["kv_len"], g["tree_offsets"], g["tree_parent"], scale)
    o = out.float().cpu().numpy()
    assert np.isfinite(o).all()
    assert np.abs(o - ref).max() <= BF16_TOL


@pytest.mark.parametrize("nq", ["1", "2", "cs2", "cs4", "2cs2"])
@pytest.mark.parametrize("pad", ["nan", "inf"])
def test_attn_bf16_nan_in_tree_padding(ada, nq, pad):
    """Tree tiles are loaded 64 rows at a time from the request's first row: the
    rows past K_i belong to the next request or to the caller's padding past
    tree_offsets[n] (e.g. a budget-sized torch.empty buffer).  NaN/Inf there
    must not reach any output (P is 0 there, but 0 * NaN = NaN in the PV MMA).
    K_i around the 64-row tile edges: 63, 64, 65, 127, 128."""
    sched = _sched(nq)
    sizes = [63, 64, 65, 127, 128, 1, 191, 256]
    w = _attn_case((sizes, [70, 0, 129, 64, 5, 33, 64, 1], 8, 2, 128, 64, "random", 1.0), True, 91)
    scale = np.float32(1.0 / np.sqrt(128))
    ref, ref_lse = oracle_attn(w, scale)
    R = int(w["tree_offsets"][-1])
    bad = np.float32(np.nan if pad == "nan" else np.inf)
    extra = 200  # budget-sized buffers: padding rows past tree_offsets[n]
    g = workload_to_device(w, torch.bfloat16)
    for k in ("q", "k_tree", "v_tree"):
        t = g[k]
        big = torch.full((R + extra,) + tuple(t.shape[1:]), float(bad), dtype=t.dtype, device=t.device)
        big[:R] = t
        g[k] = big
    par = torch.zeros(R + extra, dtype=torch.int32, device="cuda")
    par[:R] = g["tree_parent"]
    ws = ada.Workspace(256)
    out, lse = ada.tree_verify_attn(g["q"], g["k_tree"], g["v_tree"], g["k_cache"], g["v_cache"], g["page_table"],
                                    g["kv_len"], g["tree_offsets"], par, scale, want_lse=True, workspace=ws, schedule=sched)
    assert ada.check_device_error(ws)[0] == 0
    o = out[:R].float().cpu().numpy()
    assert np.isfinite(o).all()
    assert np.abs(o - ref).max() <= BF16_TOL
    assert np.abs(lse[:R].cpu().numpy() - ref_lse).max() <= BF16_TOL


def test_accept_records_vs_oracle(ada):
    """The multi-GPU record phases compared with the oracle directly (not with
    the fused GPU path): WALK_RECORDS over request shards == oracle.accept_walk
    row by row, COMMIT_RECORDS == oracle.commit byte for byte."""
    rng = np.random.default_rng(17)
    for n, world in ((45, 4), (8, 3), (1, 2)):
        X = _accept_inputs(rng, n, 40, dtype="bf16")
        mp = 24
        s = (n + world - 1) // world
        rec = torch.full((world * s, 2 + mp), -9, dtype=torch.int32, device="cuda")
        for r in range(world):
            b, e = min(n, r * s), min(n, r * s + s)
            ada.accept_tokens(ada.AS_ACCEPT_WALK_RECORDS, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                              target_tokens=dev(X["tgt"]), max_path=mp, req_range=(b, e), accept_path=rec)
        ref = oracle.accept_walk(X["to"], X["par"], X["toks"], target_tokens=X["tgt"], max_path=mp)
        got = rec.cpu().numpy()
        np.testing.assert_array_equal(got[:n, 0], ref["accept_len"])
        np.testing.assert_array_equal(got[:n, 1], ref["bonus_token"])
        np.testing.assert_array_equal(got[:n, 2:], ref["accept_path"])
        kc_g, vc_g, kl_g = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16), dev(X["kv_len"])
        kl_out = torch.full_like(kl_g, -1)
        res = ada.accept_tokens(ada.AS_ACCEPT_COMMIT_RECORDS, dev(X["to"]), max_path=mp, accept_path=rec,
                                k_tree=dev(X["kt"], torch.bfloat16), v_tree=dev(X["vt"], torch.bfloat16),
                                k_cache=kc_g, v_cache=vc_g, page_table=dev(X["table"]), kv_len=kl_g,
                                kv_len_out=kl_out, n_tree_rows=int(X["to"][-1]))
        assert ada.check_device_error(res["workspace"])[0] == 0
        to_bits = lambda a: bf16_bits(torch.from_numpy(a).to(torch.bfloat16))
        kc, vc, kt, vt = (to_bits(X[k]) for k in ("kc", "vc", "kt", "vt"))
        kl = X["kv_len"].copy()
        assert oracle.commit(X["to"], ref["accept_len"], ref["accept_path"], kt, vt, kc, vc, X["table"], kl) == 0
        np.testing.assert_array_equal(kl_out.cpu().numpy(), kl)
        np.testing.assert_array_equal(bf16_bits(kc_g).view(np.uint8), kc.view(np.uint8))
        np.testing.assert_array_equal(bf16_bits(vc_g).view(np.uint8), vc.view(np.uint8))


def test_dist_accept_and_commit_single_rank_nccl(ada):
    """paper_2501_12162_b200.dist.accept_and_commit on a single-rank NCCL group,
    eagerly and replayed from a captured CUDA graph (the static record buffer of
    ShardedAccept): equals FUSED and the oracle."""
    import torch.distributed as tdist
    from paper_2501_12162_b200.dist import ShardedAccept, accept_and_commit
    created = False
    if not tdist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        created = True
    try:
        rng = np.random.default_rng(19)
        n = 33
        X = _accept_inputs(rng, n, 30, dtype="bf16")
        kt, vt = dev(X["kt"], torch.bfloat16), dev(X["vt"], torch.bfloat16)
        args = lambda kc, vc: (dev(X["to"]), dev(X["par"]), dev(X["toks"]), kt, vt, kc, vc, dev(X["table"]),
                               dev(X["kv_len"]))
        ref = oracle.accept_walk(X["to"], X["par"], X["toks"], target_tokens=X["tgt"], max_path=24)
        kc1, vc1 = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16)
        rec = accept_and_commit(None, *args(kc1, vc1), max_path=24, target_tokens=dev(X["tgt"]))
        np.testing.assert_array_equal(rec[:n, 0].cpu().numpy(), ref["accept_len"])
        np.testing.assert_array_equal(rec[:n, 2:].cpu().numpy(), ref["accept_path"])
        kc0, vc0, kl0 = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16), dev(X["kv_len"])
        ada.accept_tokens(ada.AS_ACCEPT_FUSED, dev(X["to"]), dev(X["par"]), dev(X["toks"]),
                          target_tokens=dev(X["tgt"]), max_path=24, k_tree=kt, v_tree=vt, k_cache=kc0, v_cache=vc0,
                          page_table=dev(X["table"]), kv_len=kl0)
        assert torch.equal(kc1, kc0) and torch.equal(vc1, vc0)
        # captured: static inputs, static record buffer, replayed
        sh = ShardedAccept()
        a = args(dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16))
        tgt = dev(X["tgt"])
        klo = torch.empty_like(a[8])
        sh(*a, max_path=24, target_tokens=tgt, kv_len_out=klo)  # warm-up (NCCL communicator, attributes)
        torch.cuda.synchronize()
        kc2, vc2 = dev(X["kc"], torch.bfloat16), dev(X["vc"], torch.bfloat16)
        a = a[:5] + (kc2, vc2) + a[7:]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            sh(*a, max_path=24, target_tokens=tgt, kv_len_out=klo)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(kc2, kc0) and torch.equal(vc2, vc0) and torch.equal(klo, kl0)
        np.testing.assert_array_equal(sh.records[:n, 1].cpu().numpy(), ref["bonus_token"])
    finally:
        if created:
            tdist.destroy_process_group()


@pytest.mark.parametrize("cfg,shape", [("c2", "auto"), ("c3", "auto"), ("c4", "auto"), ("c5", "auto"),
                                       ("c4", "cs4"), ("c4", "2"), ("c5", "cs2"), ("c3", "cs2"), ("c4", "2cs2"),
                                       ("c5", "2cs2")])
def test_attn_bf16_full_size_sampled(ada, cfg, shape):
    """BASELINE full sizes in the launch bench.py times; the oracle checks sampled
    requests (all their heads).  The oracle's trees come from the oracle's own
    select on the same forest (asserted bit-identical to the GPU's)."""
    import bench
    W = bench.make_workload(cfg, device="cuda", seed_salt=5)
    W["schedule"] = ada.parse_schedule(_sched(shape))  # the CTA shape under test (None: the library's choice)
    bench.run_select(W)
    out = bench.run_attention(W)
    torch.cuda.synchronize()
    F, c = W["host"], W["c"]
    ref_sel = oracle.select_literal(F["cand_offsets"], F["cand_parent"], F["cand_prob"], W["A"], c["d"], c["n_max"],
                                    c["budget"])
    used = int(ref_sel["tree_offsets"][-1])
    np.testing.assert_array_equal(W["sel"]["tree_offsets"].cpu().numpy(), ref_sel["tree_offsets"])
    np.testing.assert_array_equal(W["sel"]["tree_parent"].cpu().numpy()[:used], ref_sel["tree_parent"])
    to = ref_sel["tree_offsets"]
    # 16 spread requests plus the largest tree and the longest prefix
    reqs = sorted(set(W["sample_requests"]) | {int(np.argmax(np.diff(to))), int(np.argmax(W["kv_len_host"]))})
    kc, vc = W["pools"][W["pool_idx"]]
    w = dict(q=W["q"].float().cpu().numpy(), k_tree=W["k_tree"].float().cpu().numpy(),
             v_tree=W["v_tree"].float().cpu().numpy(), tree_offsets=to,
             tree_parent=np.concatenate([ref_sel["tree_parent"], np.zeros(W["R"] - used, np.int32)]),
             page_table=W["table_host"], kv_len=W["kv_len_host"])
    pt = W["table_host"][reqs]
    pages = np.unique(pt[pt >= 0])
    idx = torch.from_numpy(pages).cuda()
    kfull = np.zeros((W["n_pages"],) + tuple(kc.shape[1:]), np.float32)
    vfull = np.zeros_like(kfull)
    kfull[pages] = kc.index_select(0, idx).float().cpu().numpy()
    vfull[pages] = vc.index_select(0, idx).float().cpu().numpy()
    w["k_cache"], w["v_cache"] = kfull, vfull
    rows, ref, _ = oracle_attn(w, np.float32(W["sm_scale"]), requests=reqs)
    got = out[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    assert np.abs(got - ref).max() <= BF16_TOL


# --------------------------------------------------------------------------- NEXT-2: iteration graph
def test_iteration_graph_replay_equals_eager(ada):
    """select -> attention -> accept captured once and replayed == the same
    library calls made eagerly (bit-exact: same kernels, same inputs)."""
    import bench
    from paper_2501_12162_b200.iteration import IterationGraph, IterationShape
    W = bench.make_workload("c2", "cuda", seed_salt=11)
    c = W["c"]
    N = int(W["cand_offsets"][-1])
    kc, vc = W["pools"][0]
    shape = IterationShape(W["n"], N, c["d"], c["n_max"], W["R"], W["n_q"], W["n_kv"], W["D"], kc.shape[0],
                           W["page_size"], W["page_table"].shape[1], W["max_path"])
    it = IterationGraph(shape, W["sm_scale"])
    for k, src in (("cand_offsets", W["cand_offsets"]), ("cand_parent", W["cand_parent"]),
                   ("cand_prob", W["cand_prob"]), ("cand_token", W["cand_token"]),
                   ("slo_deficit", W["slo_deficit"]), ("q", W["q"]), ("k_tree", W["k_tree"]),
                   ("v_tree", W["v_tree"]), ("target_tokens", W["target_tokens"]), ("k_cache", kc),
                   ("v_cache", vc), ("page_table", W["page_table"]), ("kv_len", W["kv_len"])):
        it.inputs[k].copy_(src)
    it.capture()
    it.inputs["k_cache"].copy_(kc)  # the capture's warm-up committed into the cache copy
    it.inputs["v_cache"].copy_(vc)
    out = it.replay()
    torch.cuda.synchronize()
    # eager reference through the bench's wrappers (same library calls)
    W["pool_idx"] = 0
    bench.run_select(W)
    ref = bench.run_attention(W)
    bench.run_accept(W)
    torch.cuda.synchronize()
    for k in ("tree_offsets", "tree_parent", "tree_src", "tree_token", "slo_count"):
        n = out[k].numel()
        assert torch.equal(out[k], W["sel"][k][:n]), k
    used = int(out["tree_offsets"][-1])
    assert torch.equal(out["out"][:used], ref[:used])
    for k in ("accept_len", "accept_path", "bonus_token"):
        assert torch.equal(out[k], W["acc"][k]), k
    assert torch.equal(out["kv_len_out"], W["kv_len_out"])


# --------------------------------------------------------------------------- NEXT-3(a) sampling
@pytest.mark.parametrize("rows,vocab,dtype,inv_t", [(37, 1000, "f32", 1.0), (19, 4099, "bf16", 0.7),
                                                    (5, 7, "f32", 2.0), (300, 64, "bf16", 0.0),
                                                    (4, 128256, "bf16", 1.0), (3, 128256, "f32", 0.6)])
def test_sample_tokens_bit_exact(ada, rows, vocab, dtype, inv_t):
    """as_sample_tokens == oracle.sampling.sample_rows token for token (R23
    fixes every fp32 operation); ragged vocabularies take the scalar path."""
    from oracle import sampling
    rng = np.random.default_rng(rows * 7 + vocab)
    lg = rng.normal(0.0, 3.0, (rows, vocab)).astype(np.float32)
    lg[0, : min(vocab, 5)] = 4.0  # exact ties in the logits
    t = torch.from_numpy(lg)
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
        lg = t.float().numpy()
    seed, offset = 0x1234_5678_9ABC + rows, vocab * 3
    got, ws = ada.sample_tokens(t.cuda(), np.float32(inv_t), seed, offset)
    assert ada.check_device_error(ws)[0] == 0
    want = sampling.sample_rows(lg, np.float32(inv_t), seed, offset)
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_stochastic_walk_with_sampled_targets(ada):
    """The stochastic walk (R13) end to end on the GPU: per-node target samples
    from as_sample_tokens feed as_accept_tokens; equals the oracle walk driven by
    the oracle's samples."""
    from oracle import sampling
    rng = np.random.default_rng(8)
    n, V = 12, 50
    sizes = rng.integers(1, 20, n)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    par = np.concatenate([[0] + [int(rng.integers(0, j)) for j in range(1, k)] for k in sizes]).astype(np.int32)
    tok = rng.integers(0, 4, offs[-1]).astype(np.int32)  # tiny alphabet: many matches
    lg = rng.normal(0.0, 1.0, (offs[-1], V)).astype(np.float32)
    lg[:, :4] += 3.0
    samp, _ = ada.sample_tokens(torch.from_numpy(lg).cuda(), 1.0, 77, 0)
    want_samp = sampling.sample_rows(lg, np.float32(1.0), 77, 0)
    np.testing.assert_array_equal(samp.cpu().numpy(), want_samp)
    max_path = int(sizes.max()) + 1
    out = ada.accept_tokens(ada.AS_ACCEPT_WALK_ONLY, dev(offs), dev(par), dev(tok), target_tokens=samp,
                            max_path=max_path, n_tree_rows=int(offs[-1]))
    ref = oracle.accept_walk(offs, par, tok, target_tokens=want_samp, max_path=max_path)
    assert ref["status"] == 0
    np.testing.assert_array_equal(out["accept_path"].cpu().numpy(), ref["accept_path"])
    np.testing.assert_array_equal(out["accept_len"].cpu().numpy(), ref["accept_len"])
    np.testing.assert_array_equal(out["bonus_token"].cpu().numpy(), ref["bonus_token"])


# --------------------------------------------------------------------------- NEXT-3(b) MSS
def _mss_dev(W):
    return (dev(W["tree_offsets"]), dev(W["tree_parent"]), dev(W["tree_tokens"]), dev(W["p"]), dev(W["q"]),
            dev(W["uni"]), dev(W["bonus_uni"]))


def _mss_cases():
    return [  # (sizes, vocab, shape, drift, dup)
        ([1, 2, 9, 17, 40], 1000, "random", 0.5, False),
        ([33, 5, 64], 4099, "random", 1.5, False),       # ragged vocab: scalar loads
        ([12, 12, 12], 7, "star", 0.3, False),            # vocab < one thread chunk
        ([30, 30], 2000, "star", 2.0, True),              # many equal siblings, many rejections
        ([20, 20, 20], 3000, "chain", 0.1, False),        # target ~ draft: long accepted chains
        ([256, 100], 512, "random", 1.0, True),           # AS_MAX_TREE nodes
    ]


@pytest.mark.parametrize("ci", range(6))
def test_mss_all_nodes_vs_oracle(ada, ci):
    """as_mss_verify(ALL_NODES): every node's emitted token equals oracle/mss.py's
    (R25); a difference is allowed only where the oracle's decision margin says
    the fp64 sums' association can decide it (< 1e-12 relative)."""
    from oracle import mss
    sizes, V, shape, drift, dup = _mss_cases()[ci]
    W = synth.mss_workload(np.random.default_rng(100 + ci), sizes, V, drift=drift, shape=shape, dup_tokens=dup)
    _, emitted, ws = ada.mss_verify(*_mss_dev(W), mode=ada.AS_MSS_ALL_NODES)
    assert ada.check_device_error(ws)[0] == 0
    want, margin = mss.mss_tokens(W["tree_offsets"], W["tree_parent"], W["tree_tokens"], W["p"], W["q"], W["uni"],
                                  W["bonus_uni"])
    got = emitted.cpu().numpy()
    bad = np.nonzero(got != want)[0]
    assert all(margin[b] < 1e-12 for b in bad), [(int(b), int(got[b]), int(want[b]), margin[b]) for b in bad[:5]]
    assert len(bad) <= max(1, len(got) // 100)


@pytest.mark.parametrize("ci", range(6))
def test_mss_walk_records_vs_oracle(ada, ci):
    """as_mss_verify(WALK): the accept records {len, bonus, path} equal
    oracle mss_walk's; emitted holds the path nodes' tokens and -1 elsewhere."""
    from oracle import mss
    sizes, V, shape, drift, dup = _mss_cases()[ci]
    W = synth.mss_workload(np.random.default_rng(200 + ci), sizes, V, drift=drift, shape=shape, dup_tokens=dup)
    mp = max(sizes) + 1
    rec, emitted, ws = ada.mss_verify(*_mss_dev(W), max_path=mp, mode=ada.AS_MSS_WALK)
    assert ada.check_device_error(ws)[0] == 0
    ref = mss.mss_walk(W["tree_offsets"], W["tree_parent"], W["tree_tokens"], W["p"], W["q"], W["uni"],
                       W["bonus_uni"], mp)
    rec = rec.cpu().numpy()
    em = emitted.cpu().numpy()
    for i in range(len(sizes)):
        if ref["margin"][i] < 1e-12 and (rec[i, 0] != ref["accept_len"][i] or rec[i, 1] != ref["bonus_token"][i]):
            continue  # a decision at the fp64 association tie (see test_mss_all_nodes_vs_oracle)
        assert rec[i, 0] == ref["accept_len"][i], i
        assert rec[i, 1] == ref["bonus_token"][i], i
        np.testing.assert_array_equal(rec[i, 2:], ref["accept_path"][i])
        o = int(W["tree_offsets"][i])
        path = [int(x) for x in ref["accept_path"][i][: ref["accept_len"][i]]]
        for k in range(sizes[i]):
            if k not in path:
                assert em[o + k] == -1
        # the emitted token of a path node is the next path node's draft token, or the bonus
        for a, b in zip(path, path[1:] + [None]):
            assert em[o + a] == (W["tree_tokens"][o + b] if b is not None else ref["bonus_token"][i])


def test_mss_degenerate_rows(ada):
    """Closed cases: q = p accepts the first child whenever p(x) > 0 (r N q <= p
    with N = 1 up to rounding -- checked against the oracle); a one-hot target
    emits its token; a child whose token has p = 0 is always rejected; a
    root-only tree samples the bonus from p."""
    from oracle import mss
    rng = np.random.default_rng(5)
    V = 600
    sizes = [4, 4, 1, 6]
    W = synth.mss_workload(rng, sizes, V, shape="star")
    W["q"][:4] = W["p"][:4]                           # request 0: q == p
    W["p"][4:8] = 0.0
    W["p"][4:8, 17] = 1.0                             # request 1: one-hot target at token 17
    W["tree_tokens"][5] = 17
    W["p"][9:15, :] = W["p"][9:15, :]
    W["p"][9, W["tree_tokens"][10:15]] = 0.0          # request 3: every child's token has p = 0
    _, emitted, ws = ada.mss_verify(*_mss_dev(W), mode=ada.AS_MSS_ALL_NODES)
    assert ada.check_device_error(ws)[0] == 0
    got = emitted.cpu().numpy()
    want, _ = mss.mss_tokens(W["tree_offsets"], W["tree_parent"], W["tree_tokens"], W["p"], W["q"], W["uni"],
                             W["bonus_uni"])
    np.testing.assert_array_equal(got, want)
    assert got[0] == W["tree_tokens"][1]              # q == p: first child accepted
    assert got[4] == 17                               # one-hot
    assert got[9] not in set(W["tree_tokens"][10:15].tolist())


def test_mss_walk_then_commit_vs_oracle(ada):
    """MSS walk records -> as_accept_tokens(COMMIT_RECORDS): the KV cache after
    the commit equals oracle.commit of the oracle walk's paths, byte for byte."""
    from oracle import mss
    rng = np.random.default_rng(31)
    sizes = [9, 14, 3, 20]
    n = len(sizes)
    W = synth.mss_workload(rng, sizes, 700, drift=0.3)
    R = int(W["tree_offsets"][-1])
    mp = max(sizes) + 1
    n_kv, d, ps = 2, 64, 16
    kv_len = rng.integers(0, 40, n).astype(np.int32)
    pt, num_pages = synth.paged_kv(rng, kv_len, ps, extra_slots=mp)
    kt = rng.normal(size=(R, n_kv, d)).astype(np.float32)
    vt = rng.normal(size=(R, n_kv, d)).astype(np.float32)
    kc = rng.normal(size=(num_pages, n_kv, ps, d)).astype(np.float32)
    vc = rng.normal(size=(num_pages, n_kv, ps, d)).astype(np.float32)
    rec, _, ws = ada.mss_verify(*_mss_dev(W), max_path=mp, mode=ada.AS_MSS_WALK)
    g_kc, g_vc, g_len = dev(kc), dev(vc), dev(kv_len)
    res = ada.accept_tokens(ada.AS_ACCEPT_COMMIT_RECORDS, dev(W["tree_offsets"]), max_path=mp, accept_path=rec,
                            k_tree=dev(kt), v_tree=dev(vt), k_cache=g_kc, v_cache=g_vc, page_table=dev(pt),
                            kv_len=g_len, n_tree_rows=R)
    assert ada.check_device_error(res["workspace"])[0] == 0
    ref = mss.mss_walk(W["tree_offsets"], W["tree_parent"], W["tree_tokens"], W["p"], W["q"], W["uni"],
                       W["bonus_uni"], mp)
    kl = kv_len.copy()
    assert oracle.commit(W["tree_offsets"], ref["accept_len"], ref["accept_path"], kt, vt, kc, vc, pt, kl) == 0
    np.testing.assert_array_equal(g_len.cpu().numpy(), kl)
    np.testing.assert_array_equal(g_kc.cpu().numpy(), kc)
    np.testing.assert_array_equal(g_vc.cpu().numpy(), vc)


def test_mss_llama_vocab_sampled(ada):
    """|V| = 128 256 (the bench's vocabulary, one 8-CTA cluster per request):
    walk records of 3 requests vs the oracle."""
    from oracle import mss
    sizes = [32, 8, 1]
    W = synth.mss_workload(np.random.default_rng(77), sizes, synth.LLAMA3_VOCAB, drift=0.4, shape="random")
    rec, _, ws = ada.mss_verify(*_mss_dev(W), max_path=33, mode=ada.AS_MSS_WALK)
    assert ada.check_device_error(ws)[0] == 0
    ref = mss.mss_walk(W["tree_offsets"], W["tree_parent"], W["tree_tokens"], W["p"], W["q"], W["uni"],
                       W["bonus_uni"], 33)
    rec = rec.cpu().numpy()
    np.testing.assert_array_equal(rec[:, 0], ref["accept_len"])
    np.testing.assert_array_equal(rec[:, 1], ref["bonus_token"])
    np.testing.assert_array_equal(rec[:, 2:], ref["accept_path"])
