#!/usr/bin/env python
"""bench.py -- AdaServe hot path (select -> tree-verify attention -> accept+commit)
on B200.  Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (KV-head sharding, NCCL all-gather)

Metric (BASELINE.json): verified tree tokens/sec (sum_i K_i per step / step time)
and the attention kernel's HBM GB/s as a fraction of the measured HBM peak.
A step = one pass of the whole hot path over one batch: as_select_trees ->
as_tree_verify_attn (one layer) -> as_accept_tokens (walk + KV commit), plus at
N>1 the all-gather of accept records.  Inputs are resident in HBM; accept
writes the advanced prefix lengths out of place (kv_len_out), so every step
verifies the same workload with nothing but the hot path in the timed region.

The only place outside tests/ that touches oracle/ is the `cpu_baseline` leg
and `--impl reference`, which time the CPU oracle as it stands on this host.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

# --------------------------------------------------------------------------- configs (BASELINE.json)
CONFIGS = {
    "c1": dict(desc="1 request, 8-node speculation tree, 1 layer, 4 heads x head_dim 64, 128-token KV prefix, fp32",
               n_req=1, d=3, w=3, sigma=(1.0, 4.0), A="c1", n_max=7, budget=8, L=128, n_q=4, n_kv=4, head_dim=64,
               page_size=16, dtype="f32"),
    "c2": dict(desc="Llama-3-8B shapes (32 q / 8 kv heads, d=128), 64 requests, 32-node trees, 2k-token paged KV, "
                    "bf16", n_req=64, d=8, w=8, sigma=(1.0, 4.0), A=9.0, n_max=31, budget=2048, L=2048, n_q=32,
               n_kv=8, head_dim=128, page_size=64, dtype="bf16"),
    "c3": dict(desc="mixed-SLO batch: 256 requests, per-request trees 4-64 under a 4096-token global budget, "
                    "Llama-3-8B shapes, 2k KV (assumed)", n_req=256, d=8, w=8, sigma=(1.0, 8.0), A="mix", n_max=63,
               budget=4096, L=2048, n_q=32, n_kv=8, head_dim=128, page_size=64, dtype="bf16"),
    "c4": dict(desc="Llama-3-70B shapes (64 q / 8 kv heads), 128 requests, 64-node trees, 2k KV (assumed)",
               n_req=128, d=8, w=8, sigma=(1.0, 4.0), A=9.0, n_max=63, budget=8192, L=2048, n_q=64, n_kv=8,
               head_dim=128, page_size=64, dtype="bf16"),
    "c5": dict(desc="long-context stress: 32 requests, 32k-token KV prefixes, 64-node trees, Llama-3-8B shapes",
               n_req=32, d=8, w=8, sigma=(1.0, 4.0), A=9.0, n_max=63, budget=2048, L=32768, n_q=32, n_kv=8,
               head_dim=128, page_size=64, dtype="bf16"),
    # the c3 batch verify-only -- sizes K_i = 4 + floor(61 u^4) trimmed to sum <= 4096,
    # random recursive trees of depth <= 8, given (no select in the step)
    "c3b": dict(desc="c3 verify-only: 256 requests, fixed sizes K = 4 + floor(61 u^4) (sum <= 4096), random "
                     "recursive trees of depth <= 8, Llama-3-8B shapes, 2k KV; step = attention + accept",
                n_req=256, d=8, w=8, sigma=(1.0, 8.0), A="mix", n_max=63, budget=4096, L=2048, n_q=32, n_kv=8,
                head_dim=128, page_size=64, dtype="bf16", verify_only=True),
}
CONFIG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4, "c3b": 2}
# requests of the bounded CPU-oracle sample (cpu_baseline and the --impl reference arm alike)
ORACLE_SAMPLE_REQ = {"c1": 1, "c2": 64, "c3": 64, "c3b": 64, "c4": 16, "c5": 2}
METRIC = "verified tree tokens/sec and attn HBM GB/s (% roofline) at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# --------------------------------------------------------------------------- workload
def make_workload(cfg_name, device="cuda", seed_salt=0, rank=0, world=1, engine="ours"):
    """Synthetic inputs with the shapes of BASELINE config `cfg_name`.
    KV-head sharding: this rank holds kv heads [rank*n_kv/world, (rank+1)*n_kv/world).
    engine="ours" builds the CUDA-path buffers; engine="oracle" (the --impl
    reference arm, CPU only) builds host tensors and never touches the library."""
    c = dict(CONFIGS[cfg_name])
    rng = synth.rng_for(CONFIG_INDEX[cfg_name], seed_salt)
    n = c["n_req"]
    F = synth.beam_forest(rng, n, c["d"], c["w"], *c["sigma"])
    if c["A"] == "mix":
        A = synth.slo_mix(rng, n)
    elif c["A"] == "c1":
        A = np.array([0.5])
    else:
        A = np.full(n, float(c["A"]))
    assert c["n_kv"] % world == 0, "KV-head sharding needs n_kv % world == 0"
    n_kv = c["n_kv"] // world
    G = c["n_q"] // c["n_kv"]
    n_q = n_kv * G
    D = c["head_dim"]
    ps = c["page_size"]
    kv_len = np.full(n, c["L"], np.int32)
    table, n_pages = synth.paged_kv(rng, kv_len, ps, extra_slots=c["d"] + 1,
                                    permute=os.environ.get("AS_BENCH_CONTIGUOUS_PAGES") != "1")
    R = c["budget"]  # tree rows allocated = budget (upper bound of sum K_i)
    dt = torch.float32 if c["dtype"] == "f32" else torch.bfloat16
    gen = torch.Generator(device=device).manual_seed(synth.SEED_BASE + 17 * CONFIG_INDEX[cfg_name] + 1000 * seed_salt
                                                     + 7919 * rank)
    kv_bytes = 2 * n_pages * n_kv * ps * D * (4 if dt == torch.float32 else 2)
    n_pools = 1 if kv_bytes >= 3 * L2_BYTES else int(math.ceil(3 * L2_BYTES / kv_bytes))
    if cfg_name == "c1":
        n_pools = 1

    def rnd(*shape):
        return torch.randn(*shape, generator=gen, device=device, dtype=torch.float32).to(dt)

    pools = [(rnd(n_pages, n_kv, ps, D), rnd(n_pages, n_kv, ps, D)) for _ in range(n_pools)]
    W = dict(cfg=cfg_name, c=c, host=F, A=A, n=n, n_q=n_q, n_kv=n_kv, D=D, page_size=ps, R=R, dtype=dt,
             sm_scale=float(np.float32(1.0 / math.sqrt(D))), rank=rank, world=world, n_pools=n_pools,
             kv_bytes=kv_bytes, pools=pools, pool_idx=0, device=device, kv_len_host=kv_len, table_host=table,
             n_pages=n_pages)
    W["cand_offsets"] = torch.from_numpy(F["cand_offsets"]).to(device)
    W["cand_parent"] = torch.from_numpy(F["cand_parent"]).to(device)
    W["cand_prob"] = torch.from_numpy(F["cand_prob"]).to(device)
    W["cand_token"] = torch.from_numpy(F["cand_token"]).to(device)
    W["slo_deficit"] = torch.from_numpy(np.ascontiguousarray(A, np.float64)).to(device)
    W["page_table"] = torch.from_numpy(table).to(device)
    # kv_len is the committed prefix the step reads; accept writes the new
    # lengths to kv_len_out (as_accept_tokens' out-of-place form), so every
    # replayed step verifies the same workload without a restore copy.
    W["kv_len"] = torch.from_numpy(kv_len).to(device)
    W["kv_len_out"] = torch.empty_like(W["kv_len"])
    W["q"] = rnd(R, n_q, D)
    W["k_tree"] = rnd(R, n_kv, D)
    W["v_tree"] = rnd(R, n_kv, D)
    W["out"] = torch.empty_like(W["q"])
    # parity sample of the full-size test: 16 requests spread over the batch
    W["sample_requests"] = sorted(set(np.linspace(0, n - 1, min(n, 16)).round().astype(int).tolist()))
    W["max_path"] = c["d"] + 1
    if engine == "oracle":
        import oracle  # reference arm only
        sel = oracle.select_literal(F["cand_offsets"], F["cand_parent"], F["cand_prob"], A, c["d"], c["n_max"],
                                    c["budget"])
        _set_targets(W, sel["tree_offsets"], sel["tree_src"])
        if c.get("verify_only"):
            _set_given_trees(W, synth.rng_for(CONFIG_INDEX[cfg_name], 77 + seed_salt))
        return W
    import paper_2501_12162_b200 as ada
    W["ada"] = ada
    N = int(F["cand_offsets"][-1])
    W["ws_select"] = ada.Workspace(ada.select_workspace_size(n, N), device)
    W["ws_attn"] = ada.Workspace(ada.attn_workspace_size(1, n, R, n_q, D, c["L"]), device)
    W["ws_accept"] = ada.Workspace(ada.accept_workspace_size(R), device)
    dev = torch.device(device)
    W["sel"] = dict(tree_offsets=torch.empty(n + 1, dtype=torch.int32, device=dev),
                    tree_parent=torch.zeros(R, dtype=torch.int32, device=dev),
                    tree_src=torch.zeros(R, dtype=torch.int32, device=dev),
                    tree_depth=torch.zeros(R, dtype=torch.int32, device=dev),
                    tree_token=torch.zeros(R, dtype=torch.int32, device=dev),
                    slo_count=torch.empty(n, dtype=torch.int32, device=dev))
    W["acc"] = dict(accept_len=torch.empty(n, dtype=torch.int32, device=dev),
                    accept_path=torch.empty((n, W["max_path"]), dtype=torch.int32, device=dev),
                    bonus_token=torch.empty(n, dtype=torch.int32, device=dev))
    # Per-node target samples (the target model's output at every tree node): the
    # trees are a deterministic function of the forest, so they are fixed once from
    # the first (GPU) selection and gathered on the host (synthetic target model).
    run_select(W)
    _set_targets(W, W["sel"]["tree_offsets"].cpu().numpy(), W["sel"]["tree_src"].cpu().numpy())
    if c.get("verify_only"):
        _set_given_trees(W, synth.rng_for(CONFIG_INDEX[cfg_name], 77 + seed_salt))
    return W


def _set_given_trees(W, rng):
    """c3b: trees given, not selected: K_i = 4 + floor(61 u^4), the
    batch trimmed (last requests first) until sum K <= budget, random recursive
    trees of depth <= 8; draft tokens random; each node's target token is one of
    its children's tokens with probability 0.6 (else random), so walks go deep."""
    n, R = W["n"], W["R"]
    sizes = 4 + np.floor(61 * rng.random(n) ** 4).astype(np.int64)
    while sizes.sum() > W["c"]["budget"]:
        sizes[np.argmax(sizes)] -= 1
    to = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    par = np.concatenate([synth.random_tree_parents(rng, int(k), max_depth=8) for k in sizes]).astype(np.int32)
    used = int(to[-1])
    tok = rng.integers(0, synth.LLAMA3_VOCAB, used).astype(np.int32)
    tgt = rng.integers(0, synth.LLAMA3_VOCAB, used).astype(np.int32)
    for i in range(n):
        o = int(to[i])
        for v in range(int(sizes[i])):
            kids = [c for c in range(v + 1, int(sizes[i])) if par[o + c] == v]
            if kids and rng.random() < 0.6:
                tgt[o + v] = tok[o + kids[int(rng.integers(0, len(kids)))]]
    dev = W["device"]
    if "sel" in W:  # the CUDA path's tree buffers (the oracle engine has none)
        W["sel"]["tree_offsets"].copy_(torch.from_numpy(to))
        W["sel"]["tree_parent"][:used].copy_(torch.from_numpy(par))
        W["sel"]["tree_token"][:used].copy_(torch.from_numpy(tok))
    t = np.zeros(R, np.int32)
    t[:used] = tgt
    W["target_tokens"] = torch.from_numpy(t).to(dev)
    W["given"] = dict(tree_offsets=to, tree_parent=par, tree_token=tok, target=tgt)
    W["tree_sizes"] = sizes.astype(np.int64)
    W["tree_tokens_total"] = used


def _set_targets(W, to, src):
    F, n, R = W["host"], W["n"], W["R"]
    used = int(to[-1])
    req = np.repeat(np.arange(n), np.diff(to))
    tgt = np.zeros(R, np.int32)
    tgt[:used] = F["cand_target"][F["cand_offsets"][req] + src[:used]]
    W["target_tokens"] = torch.from_numpy(tgt).to(W["device"])
    W["tree_sizes"] = np.diff(to)
    W["tree_tokens_total"] = used


def run_select(W):
    ada = W["ada"]
    ada.select_trees(W["cand_offsets"], W["cand_parent"], W["cand_prob"], W["slo_deficit"], W["c"]["d"],
                     W["c"]["n_max"], W["c"]["budget"], cand_token=W["cand_token"], out=W["sel"],
                     workspace=W["ws_select"])


def run_attention(W):
    ada = W["ada"]
    kc, vc = W["pools"][W["pool_idx"]]
    out, _ = ada.tree_verify_attn(W["q"], W["k_tree"], W["v_tree"], kc, vc, W["page_table"], W["kv_len"],
                                  W["sel"]["tree_offsets"], W["sel"]["tree_parent"], W["sm_scale"], out=W["out"],
                                  workspace=W["ws_attn"], schedule=W.get("schedule"))
    return out


def run_accept(W, phase=None, req_range=None):
    ada = W["ada"]
    kc, vc = W["pools"][W["pool_idx"]]
    ada.accept_tokens(ada.AS_ACCEPT_FUSED if phase is None else phase, W["sel"]["tree_offsets"],
                      W["sel"]["tree_parent"], W["sel"]["tree_token"], target_tokens=W["target_tokens"],
                      max_path=W["max_path"], k_tree=W["k_tree"], v_tree=W["v_tree"], k_cache=kc, v_cache=vc,
                      page_table=W["page_table"], kv_len=W["kv_len"], kv_len_out=W["kv_len_out"], req_range=req_range,
                      accept_len=W["acc"]["accept_len"], accept_path=W["acc"]["accept_path"],
                      bonus_token=W["acc"]["bonus_token"], n_tree_rows=W["R"], workspace=W["ws_accept"])


def run_accept_dist(W, sharded):
    """N>1: the library's multi-GPU acceptance (paper_2501_12162_b200.dist):
    WALK_RECORDS on this rank's request shard -> in-place NCCL all-gather ->
    COMMIT_RECORDS for this rank's kv heads."""
    kc, vc = W["pools"][W["pool_idx"]]
    sharded(W["sel"]["tree_offsets"], W["sel"]["tree_parent"], W["sel"]["tree_token"], W["k_tree"], W["v_tree"],
            kc, vc, W["page_table"], W["kv_len"], max_path=W["max_path"], target_tokens=W["target_tokens"],
            kv_len_out=W["kv_len_out"], n_tree_rows=W["R"], workspace=W["ws_accept"])


def attn_algorithmic_bytes(W):
    """Per launch: K and V of every (request, kv head) prefix + tree (read once),
    Q read and O written once."""
    eb = 4 if W["dtype"] == torch.float32 else 2
    D = W["D"]
    L = W["kv_len_host"].astype(np.int64)
    K = W["tree_sizes"].astype(np.int64)
    kv = int(np.sum(2 * D * eb * (L + K))) * W["n_kv"]
    qo = int(np.sum(K)) * W["n_q"] * D * eb * 2
    return kv + qo


def attn_flops(W):
    D = W["D"]
    L = W["kv_len_host"].astype(np.int64)
    K = W["tree_sizes"].astype(np.int64)
    return int(np.sum(4 * D * K * L)) * W["n_q"]


_cudart = None


def _record(ev, external):
    """Record `ev` on the current stream.  Inside CUDA-graph capture the event
    must become an event-record NODE (cudaEventRecordExternal) to be timeable."""
    global _cudart
    if not external:
        ev.record()
        return
    import ctypes
    if _cudart is None:
        _cudart = ctypes.CDLL("libcudart.so.12")
        _cudart.cudaEventRecordWithFlags.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
    rc = _cudart.cudaEventRecordWithFlags(ctypes.c_void_p(ev.cuda_event),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 1)
    if rc != 0:
        raise RuntimeError(f"cudaEventRecordWithFlags failed: {rc}")


def make_events(n):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for e in evs:  # materialise the CUDA events outside any capture
        e.record()
    torch.cuda.synchronize()
    return evs


class Step:
    """One hot-path step on the current stream; optionally records 4 events
    (before select, before attention, before accept, after accept)."""

    def __init__(self, W, dist_ctx=None):
        self.W = W
        self.dist = dist_ctx

    def __call__(self, events=None, external=False, attn_only=False):
        """events: 4 (before select/attention/accept, after accept) or, with
        attn_only, 2 (around the attention launch)."""
        W = self.W
        W["pool_idx"] = (W["pool_idx"] + 1) % W["n_pools"]
        ea = events if (events and attn_only) else None
        eb = events if (events and not attn_only) else None
        skip = os.environ.get("AS_BENCH_SKIP", "")  # ablation only (never for reported numbers)
        if eb:
            _record(eb[0], external)
        if "select" not in skip and not W["c"].get("verify_only"):
            run_select(W)
        if eb:
            _record(eb[1], external)
        if ea:
            _record(ea[0], external)
        if "attention" not in skip:
            run_attention(W)
        if ea:
            _record(ea[1], external)
        if eb:
            _record(eb[2], external)
        if "accept" in skip:
            pass
        elif self.dist is None:
            run_accept(W)
        else:
            run_accept_dist(W, self.dist)
        if eb:
            _record(eb[3], external)
        return events


def _clock_sampler_start():
    try:
        return subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
            text=True)
    except Exception:
        return None


def _clock_sampler_stop(p, dev_index):
    if p is None:
        return None
    time.sleep(0.25)
    p.terminate()
    try:
        out = p.communicate(timeout=5)[0]
    except Exception:
        return None
    sm, mx, reasons = [], [], set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in out.strip().splitlines():
        f = [x.strip() for x in line.split(",")]
        if len(f) < 9 or f[0] != str(dev_index):
            continue
        try:
            sm.append(float(f[1]))
            mx.append(float(f[2]))
        except ValueError:
            continue
        for nm, v in zip(names, f[5:9]):
            if v.lower() == "active":
                reasons.add(nm)
    if not sm:
        return None
    return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
            "samples": len(sm)}


def _traffic_from_profiles(cfg):
    p = os.path.join(ROOT, "profiles", "attn_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(cfg)
    except Exception:
        return None


# --------------------------------------------------------------------------- CPU oracle legs
def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _tree_size_summary(sizes):
    s = np.asarray(sizes, np.int64)
    edges = [1, 2, 4, 8, 16, 32, 64, 128, 257]
    hist = {f"{edges[k]}-{edges[k + 1] - 1}": int(((s >= edges[k]) & (s < edges[k + 1])).sum())
            for k in range(len(edges) - 1)}
    return {"min": int(s.min()), "p10": float(np.percentile(s, 10)), "median": float(np.median(s)),
            "p90": float(np.percentile(s, 90)), "max": int(s.max()), "mean": round(float(s.mean()), 2),
            "hist": {k: v for k, v in hist.items() if v}}


def cpu_oracle_sample(W, n_sample_req, threads):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload:
    full select (Alg. 2 literal), attention for `n_sample_req` requests, and the
    walk + commit for those requests.  Returns (tokens, seconds, description)."""
    import oracle  # test/baseline infrastructure only
    F = W["host"]
    c = W["c"]
    t0 = time.perf_counter()
    if c.get("verify_only"):  # c3b: the trees are given (no select in the step)
        gv = W["given"]
        sel = dict(tree_offsets=gv["tree_offsets"], tree_parent=gv["tree_parent"])
    else:
        sel = oracle.select_literal(F["cand_offsets"], F["cand_parent"], F["cand_prob"], W["A"], c["d"],
                                    c["n_max"], c["budget"])
    t_sel = time.perf_counter() - t0
    n = W["n"]
    reqs = list(range(min(n_sample_req, n)))
    to = sel["tree_offsets"]
    rows = np.concatenate([np.arange(to[i], to[i + 1]) for i in reqs])
    sizes = np.array([to[i + 1] - to[i] for i in reqs])
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    pt = W["table_host"][reqs]
    used = np.unique(pt[pt >= 0])
    remap = -np.ones(W["n_pages"], np.int64)
    remap[used] = np.arange(len(used))
    pt2 = np.where(pt >= 0, remap[np.maximum(pt, 0)], -1).astype(np.int32)
    idx = torch.from_numpy(used).to(W["device"])
    kc, vc = W["pools"][0]
    hk = kc.index_select(0, idx).float().cpu().numpy()
    hv = vc.index_select(0, idx).float().cpu().numpy()
    rows_t = torch.from_numpy(rows).to(W["device"])
    q = W["q"].index_select(0, rows_t).float().cpu().numpy()
    kt = W["k_tree"].index_select(0, rows_t).float().cpu().numpy()
    vt = W["v_tree"].index_select(0, rows_t).float().cpu().numpy()
    kl = W["kv_len_host"][reqs].copy()
    t0 = time.perf_counter()
    oracle.tree_attn(q, kt, vt, hk, hv, pt2, kl, offs, sel["tree_parent"][rows], np.float32(W["sm_scale"]),
                     n_threads=threads, want_lse=False)
    t_attn = time.perf_counter() - t0
    if c.get("verify_only"):
        tt = W["given"]["tree_token"][rows]
    else:
        toks = np.asarray(F["cand_token"])
        req_of = np.repeat(np.arange(len(reqs)), sizes)
        tt = toks[F["cand_offsets"][np.array(reqs)][req_of] + sel["tree_src"][rows]]
    tg = W["target_tokens"].cpu().numpy()[rows]
    t0 = time.perf_counter()
    acc = oracle.accept_walk(offs, sel["tree_parent"][rows], tt, target_tokens=tg, max_path=W["max_path"])
    oracle.commit(offs, acc["accept_len"], acc["accept_path"], kt, vt, hk, hv, pt2, kl)
    t_acc = time.perf_counter() - t0
    frac = len(reqs) / n
    secs = t_sel * frac + t_attn + t_acc
    desc = (f"oracle (C, fp64) on {len(reqs)}/{n} requests of {W['cfg']}: attention + walk/commit for those "
            f"requests, " + ("trees given (verify-only)" if c.get("verify_only") else
                             f"Alg. 2 select on the full batch pro-rated ({t_sel:.3f}s x {frac:.3f})") +
            f"; {threads} threads")
    return int(sizes.sum()), secs, desc


# --------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-spec", action="store_true", help="skip the NEXT-1 speculation-layer measurement")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / cpu legs)")
    ap.add_argument("--schedule", default="", help="attention schedule override, e.g. nq=2,cs=1,split=0 (A/B only)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return main_reference(args, rank, world)
    torch.cuda.set_device(local_rank)
    dist_ctx = None
    force_dist = os.environ.get("AS_BENCH_FORCE_DIST") == "1"  # test only: the N>1 code path on one GPU
    if world > 1 or force_dist:
        import torch.distributed as dist
        if force_dist and world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        from paper_2501_12162_b200.dist import ShardedAccept
        dist_ctx = ShardedAccept()  # default process group
    emu = int(os.environ.get("AS_BENCH_EMULATE_WORLD", "0"))  # analysis only: one rank's shard of an N-GPU run
    W = make_workload(args.config, "cuda", rank=rank, world=emu if (emu > 1 and world == 1) else world)
    if args.schedule:
        W["schedule"] = W["ada"].parse_schedule(args.schedule)
    step = Step(W, dist_ctx)
    use_graph = not args.no_graph
    for _ in range(2):  # eager warm-up (attribute setup, NCCL communicator)
        step()
    torch.cuda.synchronize()
    # Timed graph: K unrolled steps, events only around each attention launch
    # (the roofline kernel) and around the whole region.  A second graph with
    # events around every call gives the per-kernel breakdown (not the value).
    all_ev = make_events(2 * args.steps + 2)
    start, end = all_ev[-2], all_ev[-1]
    attn_ev = [all_ev[2 * k:2 * k + 2] for k in range(args.steps)]
    brk_ev = [make_events(4) for _ in range(args.steps)]
    if use_graph:
        # The whole hot path of a step is replayed from CUDA graphs.
        g_warm = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_warm):
            step()
        g_timed = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_timed):
            _record(start, True)
            for k in range(args.steps):
                step(attn_ev[k], external=True, attn_only=True)
            _record(end, True)
        g_brk = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_brk):
            for k in range(args.steps):
                step(brk_ev[k], external=True)
        for _ in range(args.warmup):
            g_warm.replay()
    else:
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler = None if args.profile else _clock_sampler_start()
    if sampler is not None:
        time.sleep(0.3)
    if use_graph:
        g_timed.replay()
    else:
        start.record()
        for k in range(args.steps):
            step(attn_ev[k], attn_only=True)
        end.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = _clock_sampler_stop(sampler, local_rank)
    total_ms = start.elapsed_time(end)
    t_attn = float(np.mean([e[0].elapsed_time(e[1]) for e in attn_ev]))
    # breakdown pass (not timed for the value)
    if use_graph:
        g_brk.replay()
    else:
        for k in range(args.steps):
            step(brk_ev[k])
    torch.cuda.synchronize()
    t_sel = float(np.mean([e[0].elapsed_time(e[1]) for e in brk_ev]))
    t_attn_b = float(np.mean([e[1].elapsed_time(e[2]) for e in brk_ev]))
    t_acc = float(np.mean([e[2].elapsed_time(e[3]) for e in brk_ev]))
    # per-step distributions: attention launches of the timed graph, whole steps of the
    # instrumented replay (select start -> accept end)
    attn_each = np.array([e[0].elapsed_time(e[1]) for e in attn_ev])
    step_each = np.array([e[0].elapsed_time(e[3]) for e in brk_ev])
    dist_stats = lambda a: {"median": round(float(np.median(a)), 4), "p10": round(float(np.percentile(a, 10)), 4),
                            "p90": round(float(np.percentile(a, 90)), 4), "n": int(len(a))}
    if world > 1:
        # max over ranks: the step and the attention launch (the roofline uses the slowest rank)
        t = torch.tensor([total_ms, t_attn], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, t_attn = float(t[0]), float(t[1])
    ms_per_step = total_ms / args.steps
    tokens = int(W["tree_tokens_total"])
    value = tokens / (ms_per_step / 1e3)

    peaks, peak_kind = _peaks()
    abytes = attn_algorithmic_bytes(W)
    aflops = attn_flops(W)
    achieved_gbs = abytes / (t_attn / 1e3) / 1e9
    achieved_tf = aflops / (t_attn / 1e3) / 1e12
    hbm_peak = float(peaks["hbm_gbs"])
    # bf16 dense peak for a kernel timed alone (burst); the kernel also reports
    # its fraction of the sustained figure.  fp32 (SIMT, c1) has no tensor bound.
    tf_peak = float(peaks.get("bf16_tflops", 1590.0))
    tf_sus = float(peaks.get("bf16_tflops_sustained", 1400.0))
    ai = aflops / abytes if abytes else 0.0
    ridge = tf_peak * 1e12 / (hbm_peak * 1e9)
    tensor_bound = W["dtype"] == torch.bfloat16 and ai > ridge
    common = {"traffic": _traffic_from_profiles(args.config),
              "kernel": "tree_attn_tc_kernel" if W["dtype"] == torch.bfloat16 else "tree_attn_simt_kernel",
              "algorithmic_bytes_per_launch": abytes, "algorithmic_flops_per_launch": aflops,
              "arith_intensity": round(ai, 1), "ridge": round(ridge, 1), "attn_ms": round(t_attn, 4),
              "hbm_gbs": round(achieved_gbs, 1), "hbm_frac": round(achieved_gbs / hbm_peak, 4),
              "tensor_tflops": round(achieved_tf, 1), "tensor_frac_burst": round(achieved_tf / tf_peak, 4),
              "tensor_frac_sustained": round(achieved_tf / tf_sus, 4), "peak_source": peak_kind}
    if tensor_bound:
        roofline = {"bound": "tensor", "achieved": round(achieved_tf, 1), "peak": tf_peak, "unit": "TFLOP/s",
                    "frac": round(achieved_tf / tf_peak, 4), **common}
    else:
        roofline = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(achieved_gbs / hbm_peak, 4), **common}

    e2e = None
    if not args.no_e2e and not args.profile:
        e2e = measure_e2e(W, step, args.steps, world)
    spec = None
    logits_mode = None
    sampling = None
    mss = None
    if rank == 0 and not args.profile and not args.no_spec:
        spec = measure_speculation(W, args.steps)
        logits_mode = measure_accept_logits(W, args.steps)
        sampling = measure_sampling(W, args.steps)
        mss = measure_mss(W, args.steps)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        threads = os.cpu_count() or 1
        n_s = ORACLE_SAMPLE_REQ[args.config]
        timed = {}
        for nth, budget_s in ((threads, 10.0), (1, 8.0)):  # all cores, then one thread
            toks_t, secs_t, reps = 0, 0.0, 0
            while (secs_t < budget_s and reps < 50) or reps == 0:
                toks, secs, desc = cpu_oracle_sample(W, n_s, nth)
                toks_t, secs_t, reps = toks_t + toks, secs_t + secs, reps + 1
            timed[nth] = (toks_t / secs_t, desc, reps, secs_t)
        v, desc, reps, secs_t = timed[threads]
        cpu = {"value": round(v, 2), "unit": "verified tree tokens/s", "cores": threads, "kind": "oracle",
               "sample": f"{desc}; repeated {reps}x", "seconds": round(secs_t, 3), "cpu_model": _cpu_model(),
               "single_thread_value": round(timed[1][0], 2), "single_thread_seconds": round(timed[1][3], 3)}
    # select, attention, accept (walk + commit at N>1, plus the NCCL all-gather); no select in c3b
    launches_per_step = (3 if world == 1 else 4) - (1 if W["c"].get("verify_only") else 0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "verified tree tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if W["dtype"] == torch.bfloat16 else "f32", "data": "synthetic (seeded; no datasets)",
            "config": {"workload": f"{args.config}: {W['c']['desc']}", "n_req": W["n"],
                       "tree_tokens": tokens, "kv_len": W["c"]["L"], "q_heads": W["c"]["n_q"],
                       "kv_heads": W["c"]["n_kv"], "head_dim": W["D"], "page_size": W["page_size"],
                       "budget": W["c"]["budget"], "tree_sizes": _tree_size_summary(W["tree_sizes"]),
                       "verify_only": bool(W["c"].get("verify_only", False)), "parallelism": f"kv-head sharding x{world}" if world > 1
                       else "1 GPU", "l2": ("inputs larger than L2: KV %.0f MiB/GPU" % (W["kv_bytes"] / 2**20))
                       if W["n_pools"] == 1 else f"{W['n_pools']} rotating KV pools (> 3x L2)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks, "graph": use_graph, "speculation": spec, "accept_logits": logits_mode,
            "sampling": sampling, "mss": mss,
            **({"emulated_shard_of_world": emu} if (emu > 1 and world == 1) else {}), **({"ablation_skip": os.environ["AS_BENCH_SKIP"]}
                                                       if os.environ.get("AS_BENCH_SKIP") else {}),
            "breakdown_ms": {"select": round(t_sel, 4), "attention": round(t_attn_b, 4), "accept_commit": round(t_acc, 4),
                             "note": "separate instrumented replay (events around every call)"},
            "attention_tokens_per_s": round(tokens / (t_attn / 1e3), 1),
            "distribution_ms": {"attention": dist_stats(attn_each), "step": dist_stats(step_each),
                                "note": "attention: CUDA events around each launch of the timed graph; step: "
                                        "select start -> accept end in the instrumented replay"},
        }
        print(json.dumps(line), flush=True)
    if dist_ctx is not None:
        torch.distributed.destroy_process_group()


def measure_speculation(W, steps):
    """NEXT-1: one Step 1 beam layer at this config's
    shapes -- n requests x w kept nodes x |V| = 128 256 draft probabilities
    (fp32, synthetic, > L2) -> top-w per request written into a candidate
    forest.  HBM-bound: algorithmic bytes = the probabilities read once."""
    ada = W["ada"]
    c = W["c"]
    n, w, V = W["n"], c["w"], synth.LLAMA3_VOCAB
    if c["dtype"] != "bf16":
        return None
    dev = torch.device(W["device"])
    gen = torch.Generator(device=dev).manual_seed(synth.SEED_BASE + 99)
    # draft distributions as in the forest generator: softmax of
    # z ~ N(0, sigma^2) over the vocabulary, sigma ~ U(1, 4) per request
    if os.environ.get("AS_BENCH_SPEC_DIST") == "uniform":  # A/B only
        probs = torch.rand((n, w, V), generator=gen, device=dev, dtype=torch.float32)
        probs /= probs.sum(dim=-1, keepdim=True)
    else:
        sigma = torch.empty((n, 1, 1), device=dev).uniform_(1.0, 4.0, generator=gen)
        z = torch.randn((n, w, V), generator=gen, device=dev, dtype=torch.float32) * sigma
        probs = torch.softmax(z, dim=-1)
        del z
    stride = 1 + c["d"] * w
    par = torch.zeros(n * stride, dtype=torch.int32, device=dev)
    prob = torch.zeros(n * stride, dtype=torch.float32, device=dev)
    prob[::stride] = 1.0
    tok = torch.zeros(n * stride, dtype=torch.int32, device=dev)
    root = probs[:, :1, :].contiguous()
    ws = ada.beam_step(1, w, root, par, prob, tok, stride)
    for _ in range(3):
        ada.beam_step(2, w, probs, par, prob, tok, stride, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # replayed: no host launch overhead between layers
    with torch.cuda.graph(g):
        for _ in range(steps):
            ada.beam_step(2, w, probs, par, prob, tok, stride, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / steps
    nbytes = probs.numel() * 4
    peak = float(_peaks()[0]["hbm_gbs"])
    gbs = nbytes / (us * 1e-6) / 1e9
    return {"step": "beam layer (as_beam_step, layer 2)", "n_req": n, "width": w, "vocab": V,
            "draft_probs": "softmax(N(0, sigma^2)), sigma ~ U(1,4) per request, fp32",
            "layer_us": round(us, 2), "algorithmic_bytes": nbytes, "hbm_gbs": round(gbs, 1),
            "hbm_frac": round(gbs / peak, 4), "launches": 2}


def measure_accept_logits(W, steps):
    """S8 logits mode: greedy targets from per-node target logits
    [N_tree, |V| = 128 256] bf16 -- an HBM-bound argmax scan (lowest index on
    ties) -- then the walk and commit, through as_accept_tokens.  Algorithmic
    bytes = the logits read once."""
    ada = W["ada"]
    if W["dtype"] != torch.bfloat16:
        return None
    R, V = W["R"], synth.LLAMA3_VOCAB
    gen = torch.Generator(device=W["device"]).manual_seed(synth.SEED_BASE + 7)
    logits = torch.randn((R, V), generator=gen, device=W["device"], dtype=torch.float32).to(torch.bfloat16)
    kc, vc = W["pools"][W["pool_idx"]]

    def call():
        ada.accept_tokens(ada.AS_ACCEPT_FUSED, W["sel"]["tree_offsets"], W["sel"]["tree_parent"],
                          W["sel"]["tree_token"], target_logits=logits, max_path=W["max_path"], k_tree=W["k_tree"],
                          v_tree=W["v_tree"], k_cache=kc, v_cache=vc, page_table=W["page_table"],
                          kv_len=W["kv_len"], kv_len_out=W["kv_len_out"], accept_len=W["acc"]["accept_len"],
                          accept_path=W["acc"]["accept_path"], bonus_token=W["acc"]["bonus_token"],
                          n_tree_rows=R, workspace=W["ws_accept"])
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(steps):
            call()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / steps
    nbytes = int(W["tree_tokens_total"]) * V * 2
    peak = float(_peaks()[0]["hbm_gbs"])
    gbs = nbytes / (us * 1e-6) / 1e9
    del logits
    return {"step": "accept, logits mode (argmax scan + walk + commit)", "rows": int(W["tree_tokens_total"]),
            "vocab": V, "us": round(us, 2), "algorithmic_bytes": nbytes, "hbm_gbs": round(gbs, 1),
            "hbm_frac": round(gbs / peak, 4), "launches": 2}


def measure_sampling(W, steps):
    """NEXT-3(a): per-node target samples by Gumbel-max (as_sample_tokens) over
    the same [N_tree, 128 256] bf16 target logits.  ALU-bound (10 Philox rounds
    per 4 tokens, two R23 logarithms per token): reported as scored tokens/s
    against DESIGN.md's FP32-lane peak, plus the HBM fraction for context."""
    ada = W["ada"]
    if W["dtype"] != torch.bfloat16:
        return None
    R, V = W["R"], synth.LLAMA3_VOCAB
    gen = torch.Generator(device=W["device"]).manual_seed(synth.SEED_BASE + 8)
    logits = torch.randn((R, V), generator=gen, device=W["device"], dtype=torch.float32).to(torch.bfloat16)
    out = torch.empty(R, dtype=torch.int32, device=W["device"])
    ws = ada.Workspace(256, W["device"])
    for _ in range(3):
        ada.sample_tokens(logits, 1.0, 1234, 0, out=out, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for k in range(steps):
            ada.sample_tokens(logits, 1.0, 1234, k, out=out, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / steps
    toks = R * V
    nbytes = toks * 2
    peak = float(_peaks()[0]["hbm_gbs"])
    gbs = nbytes / (us * 1e-6) / 1e9
    del logits
    # issue-bound: warp instructions per scored token from the ncu capture of the
    # pruned kernel (profiles/r01/ncu_sample_c2_r01j.md: 323.9e6 / (2048 * 128256)
    # on these c2 logits -- data-dependent); peak = 148 SMs x 4 schedulers x 1 warp
    # instruction per clock at the max SM clock
    winst = 323894291 / (2048 * 128256)
    clk = float((_peaks()[0].get("sm_max_mhz") or 1965)) * 1e6
    issue_peak = 148 * 4 * clk
    achieved = toks / (us * 1e-6) * winst
    return {"step": "per-node target samples, Gumbel-max (as_sample_tokens)", "rows": R, "vocab": V,
            "us": round(us, 2), "scored_tokens_per_s": round(toks / (us * 1e-6), 1), "bound": "alu",
            "alu": {"achieved_warp_inst_per_s": round(achieved, 1), "peak_warp_inst_per_s": issue_peak,
                    "frac": round(achieved / issue_peak, 4), "warp_inst_per_token": round(winst, 4)},
            "algorithmic_bytes": nbytes, "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4), "launches": 1}


def measure_mss(W, steps):
    """NEXT-3(b): SpecInfer multi-step speculative sampling (as_mss_verify, R25)
    on this config's selected trees with |V| = 128 256 fp32 target/draft rows
    per node (q = softmax(z), z ~ N(0, sigma^2), sigma ~ U(1, 4) per node;
    p = softmax(z + 0.5 N(0, 1)); every child's token DRAWN from its parent's q).
    WALK mode reads the rows of the visited nodes only (algorithmic bytes =
    p row of every visited node + q row of every visited node with children);
    ALL_NODES reads every node's rows (HBM-bound, for context)."""
    ada = W["ada"]
    if W["dtype"] != torch.bfloat16:
        return None
    R, V, n = W["R"], synth.LLAMA3_VOCAB, W["n"]
    dv = W["device"]
    gen = torch.Generator(device=dv).manual_seed(synth.SEED_BASE + 11)
    offs = W["sel"]["tree_offsets"]
    par = W["sel"]["tree_parent"]
    sigma = torch.empty((R, 1), device=dv).uniform_(1.0, 4.0, generator=gen)
    z = torch.randn((R, V), generator=gen, device=dv) * sigma
    q = torch.softmax(z, dim=-1)
    z.add_(0.5 * torch.randn((R, V), generator=gen, device=dv))
    p = torch.softmax(z, dim=-1)
    del z
    offs_h = offs.cpu().numpy().astype(np.int64)
    U = int(offs_h[-1])  # rows in use
    par_h = par[:U].cpu().numpy().astype(np.int64)
    req = np.repeat(np.arange(n), np.diff(offs_h))
    prow = torch.from_numpy(offs_h[req] + par_h).to(dv)  # parent row of every node
    tok = torch.zeros(R, dtype=torch.int32, device=dv)
    tok[:U] = torch.multinomial(q[prow], 1, generator=gen).squeeze(1).to(torch.int32)
    uni = torch.rand(R, generator=gen, device=dv).clamp_(min=2.0 ** -24)
    bon = torch.rand(R, generator=gen, device=dv).clamp_(min=2.0 ** -24)
    mp = W["max_path"]
    rec = torch.empty((n, mp + 2), dtype=torch.int32, device=dv)
    em = torch.empty(R, dtype=torch.int32, device=dv)
    ws = W.get("mss_ws") or ada.Workspace(256, dv)  # (scripts/mss_trace.py passes a traced one)
    res = {}
    modes = ((ada.AS_MSS_WALK, "walk"), (ada.AS_MSS_ALL_NODES, "all_nodes"))
    if "mss_ws" in W:
        modes = modes[:1]
    for mode, name in modes:
        def call():
            ada.mss_verify(offs, par, tok, p, q, uni, bon, max_path=mp, mode=mode, records=rec, emitted=em,
                           workspace=ws)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(steps):
                call()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        res[name] = s.elapsed_time(e) * 1e3 / steps
        if mode == ada.AS_MSS_WALK:
            rec_h = rec.cpu().numpy()
    assert ada.check_device_error(ws)[0] == 0
    has_kids = np.zeros(U, bool)
    nonroot = np.ones(U, bool)
    nonroot[offs_h[:-1][np.diff(offs_h) > 0]] = False
    has_kids[(offs_h[req] + par_h)[nonroot]] = True
    visited = [int(offs_h[i] + rec_h[i, 2 + k]) for i in range(n) for k in range(int(rec_h[i, 0]))]
    walk_bytes = sum(V * 4 * (2 if has_kids[r] else 1) for r in visited)
    all_bytes = int(U * V * 4 + has_kids.sum() * V * 4)
    peak = float(_peaks()[0]["hbm_gbs"])
    acc = rec_h[:, 0].astype(np.float64)
    res.setdefault("all_nodes", float("nan"))
    return {"step": "SpecInfer multi-step speculative sampling (as_mss_verify)", "rows": R, "vocab": V,
            "walk_us": round(res["walk"], 2), "all_nodes_us": round(res["all_nodes"], 2),
            "mean_accept_len": round(float(acc.mean()), 3), "visited_rows": len(visited),
            "walk_algorithmic_bytes": walk_bytes, "walk_hbm_gbs": round(walk_bytes / (res["walk"] * 1e-6) / 1e9, 1),
            "walk_hbm_frac": round(walk_bytes / (res["walk"] * 1e-6) / 1e9 / peak, 4),
            "all_nodes_algorithmic_bytes": all_bytes,
            "all_nodes_hbm_frac": round(all_bytes / (res["all_nodes"] * 1e-6) / 1e9 / peak, 4),
            "inputs": "q = softmax(N(0, sigma^2)), sigma ~ U(1,4); p = softmax(z + 0.5 N(0,1)); children drawn from q",
            "launches": 1}


def measure_e2e(W, step, steps, world):
    """Same metric through the public API with HOST inputs: every step copies its
    inputs (candidate forest, A, q/k_tree/v_tree, per-node targets) from pinned
    host memory and reads the accept results back.  The copies of step k+1 run
    on a copy stream while step k computes (two device input sets, events), so
    the host link and the GPU overlap as they would in a serving loop."""
    names = ["cand_offsets", "cand_parent", "cand_prob", "cand_token", "slo_deficit", "q", "k_tree", "v_tree",
             "target_tokens"]
    host = {k: W[k].cpu().pin_memory() for k in names}
    sets = [{k: W[k] for k in names}, {k: torch.empty_like(W[k]) for k in names}]
    # accept results: the three arrays at N=1, the all-gathered record rows at N>1
    res = dict(W["acc"]) if step.dist is None else {"records": step.dist.records}
    outs = list(res)
    host_out = {k: torch.empty_like(res[k], device="cpu").pin_memory() for k in outs}
    h2d = sum(host[k].numel() * host[k].element_size() for k in names)
    d2h = sum(host_out[k].numel() * host_out[k].element_size() for k in outs)
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    ev_copied = [torch.cuda.Event(), torch.cuda.Event()]
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]

    def run(n):
        with torch.cuda.stream(copy):
            copy.wait_stream(comp)
            for k in names:
                sets[0][k].copy_(host[k], non_blocking=True)
            ev_copied[0].record(copy)
        for i in range(n):
            b = i % 2
            if i + 1 < n:  # prefetch the next step's inputs into the other set
                nb = (i + 1) % 2
                with torch.cuda.stream(copy):
                    if i >= 1:
                        copy.wait_event(ev_done[nb])  # step i-1 has finished reading that set
                    for k in names:
                        sets[nb][k].copy_(host[k], non_blocking=True)
                    ev_copied[nb].record(copy)
            comp.wait_event(ev_copied[b])
            W.update(sets[b])
            step()
            for k in outs:
                host_out[k].copy_(res[k], non_blocking=True)
            ev_done[b].record(comp)
        W.update(sets[0])

    run(2)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    run(steps)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t[0])
    v = W["tree_tokens_total"] / (ms / steps / 1e3)
    return {"value": round(v, 1), "unit": "verified tree tokens/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms / steps, 4),
            "pipelined": "H2D of step k+1 on a copy stream overlaps step k"}


def main_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands (this tier's reference arm)."""
    if rank != 0:
        return
    W = make_workload(args.config, "cpu", engine="oracle")
    threads = os.cpu_count() or 1
    # the cpu_baseline sample, shrunk for long runs so that K + W steps stay within a few minutes
    n_s = max(1, min(ORACLE_SAMPLE_REQ[args.config],
                     ORACLE_SAMPLE_REQ[args.config] * 40 // max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_oracle_sample(W, n_s, threads)
    tot_tok, tot_s = 0, 0.0
    desc = ""
    for _ in range(args.steps):
        toks, secs, desc = cpu_oracle_sample(W, n_s, threads)
        tot_tok += toks
        tot_s += secs
    value = tot_tok / tot_s
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "verified tree tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * tot_s / args.steps, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; no datasets)",
            "config": {"workload": f"{args.config}: {CONFIGS[args.config]['desc']}"},
            "cpu_baseline": {"value": round(value, 2), "unit": "verified tree tokens/s", "cores": threads,
                             "kind": "oracle", "sample": desc, "cpu_model": _cpu_model()},
            "e2e": {"value": round(value, 2), "unit": "verified tree tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
