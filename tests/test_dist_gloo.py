"""World-size-2 gloo tests (CPU) of the multi-GPU protocol's host logic:
request sharding + record packing + all-gather reproduce the single-process
walk; KV-head sharding of attention is a partition of the heads."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2501_12162_b200.dist import (all_gather_in_place, all_gather_records, head_range, pack_records,
                                        record_shard, request_range, unpack_records)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _walk_inputs(seed, n):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(1, 20, n)
    to = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    par = np.concatenate([synth.random_tree_parents(rng, int(k)) for k in sizes]).astype(np.int32)
    R = int(to[-1])
    toks = rng.integers(0, 3, R).astype(np.int32)
    tgt = rng.integers(0, 3, R).astype(np.int32)
    return to, par, toks, tgt


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    to, par, toks, tgt = _walk_inputs(5, n)
    mpth = 20
    b, e, s = request_range(n, rank, world)
    # this rank's shard of the walk (oracle stands in for the WALK_ONLY kernel)
    sub_to = (to[b:e + 1] - to[b]).astype(np.int32)
    rows = slice(int(to[b]), int(to[e]))
    r = oracle.accept_walk(sub_to, par[rows], toks[rows], target_tokens=tgt[rows], max_path=mpth)
    al = torch.zeros(n, dtype=torch.int32)
    ap = torch.zeros((n, mpth), dtype=torch.int32)
    bt = torch.zeros(n, dtype=torch.int32)
    al[b:e] = torch.from_numpy(r["accept_len"])
    ap[b:e] = torch.from_numpy(r["accept_path"])
    bt[b:e] = torch.from_numpy(r["bonus_token"])
    rec = pack_records(al, ap, bt, b, e, s)
    g = all_gather_records(rec, world)
    al2, ap2, bt2 = torch.empty_like(al), torch.empty_like(ap), torch.empty_like(bt)
    unpack_records(g, n, al2, ap2, bt2)
    full = oracle.accept_walk(to, par, toks, target_tokens=tgt, max_path=mpth)
    ok = (np.array_equal(al2.numpy(), full["accept_len"]) and np.array_equal(ap2.numpy(), full["accept_path"])
          and np.array_equal(bt2.numpy(), full["bonus_token"]))
    q.put((rank, ok))
    dist.destroy_process_group()


def _worker_records(rank, world, port, n, q):
    """The record protocol the GPU path uses (AS_ACCEPT_WALK_RECORDS ->
    in-place all_gather_into_tensor -> AS_ACCEPT_COMMIT_RECORDS), with the
    oracle standing in for the two kernels: every rank ends with every
    request's record, and committing them for this rank's kv heads equals the
    single-process commit of those heads."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    to, par, toks, tgt = _walk_inputs(9, n)
    mpth = 20
    b, e, s = request_range(n, rank, world)
    rec = torch.full((world * s, 2 + mpth), -7, dtype=torch.int32)
    sub_to = (to[b:e + 1] - to[b]).astype(np.int32)
    rows = slice(int(to[b]), int(to[e]))
    if e > b:
        r = oracle.accept_walk(sub_to, par[rows], toks[rows], target_tokens=tgt[rows], max_path=mpth)
        mine = record_shard(rec, rank, s)
        mine[:e - b, 0] = torch.from_numpy(r["accept_len"])
        mine[:e - b, 1] = torch.from_numpy(r["bonus_token"])
        mine[:e - b, 2:] = torch.from_numpy(r["accept_path"])
    all_gather_in_place(rec, rank, world)
    full = oracle.accept_walk(to, par, toks, target_tokens=tgt, max_path=mpth)
    ok = (np.array_equal(rec[:n, 0].numpy(), full["accept_len"]) and
          np.array_equal(rec[:n, 1].numpy(), full["bonus_token"]) and
          np.array_equal(rec[:n, 2:].numpy(), full["accept_path"]))
    # commit from the gathered records for this rank's heads == the full commit's head slice
    rng = np.random.default_rng(4)
    R = int(to[-1])
    n_kv, d, ps = 4, 8, 4
    kv_len = rng.integers(0, 9, n).astype(np.int32)
    table, n_pages = synth.paged_kv(rng, kv_len, ps, extra_slots=mpth + 2)
    kt = rng.standard_normal((R, n_kv, d)).astype(np.float32)
    vt = rng.standard_normal((R, n_kv, d)).astype(np.float32)
    kc = rng.standard_normal((n_pages, n_kv, ps, d)).astype(np.float32)
    vc = rng.standard_normal((n_pages, n_kv, ps, d)).astype(np.float32)
    h0, h1 = head_range(n_kv, rank, world)
    kc_all, vc_all, kl_all = kc.copy(), vc.copy(), kv_len.copy()
    oracle.commit(to, full["accept_len"], full["accept_path"], kt, vt, kc_all, vc_all, table, kl_all)
    kc_me = np.ascontiguousarray(kc[:, h0:h1])
    vc_me = np.ascontiguousarray(vc[:, h0:h1])
    kl_me = kv_len.copy()
    oracle.commit(to, rec[:n, 0].numpy().copy(), rec[:n, 2:].numpy().copy(), np.ascontiguousarray(kt[:, h0:h1]),
                  np.ascontiguousarray(vt[:, h0:h1]), kc_me, vc_me, table, kl_me)
    ok = ok and np.array_equal(kc_me, kc_all[:, h0:h1]) and np.array_equal(vc_me, vc_all[:, h0:h1])
    ok = ok and np.array_equal(kl_me, kl_all)
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(7, 2), (64, 2), (1, 2), (10, 4)])
def test_record_protocol_gloo(n, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_records, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.parametrize("n", [7, 64, 1])
def test_sharded_walk_allgather_gloo(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_head_sharding_partitions_attention():
    """Attention on each rank's kv-head shard == the matching head slice of the
    unsharded attention (oracle; bit-exact since heads are independent)."""
    rng = np.random.default_rng(3)
    w = synth.tree_workload(rng, [5, 9], [40, 17], 8, 4, 32, 16)
    full, _ = oracle.tree_attn(w["q"], w["k_tree"], w["v_tree"], w["k_cache"], w["v_cache"], w["page_table"],
                               w["kv_len"], w["tree_offsets"], w["tree_parent"], np.float32(0.2))
    world = 4
    G = 2
    for r in range(world):
        h0, h1 = head_range(4, r, world)
        sh, _ = oracle.tree_attn(w["q"][:, h0 * G:h1 * G], w["k_tree"][:, h0:h1], w["v_tree"][:, h0:h1],
                                 w["k_cache"][:, h0:h1], w["v_cache"][:, h0:h1], w["page_table"], w["kv_len"],
                                 w["tree_offsets"], w["tree_parent"], np.float32(0.2))
        np.testing.assert_array_equal(sh, full[:, h0 * G:h1 * G])
    with pytest.raises(ValueError):
        head_range(8, 0, 3)
    assert [request_range(10, r, 4)[:2] for r in range(4)] == [(0, 3), (3, 6), (6, 9), (9, 10)]
