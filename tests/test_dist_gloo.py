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
from paper_2501_12162_b200.dist import (ShardedAccept, accept_and_commit, all_gather_in_place, all_gather_records,
                                        head_range, pack_records, record_shard, request_range, unpack_records)


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


def _cpu_record_kernels(phase, tree_offsets, tree_parent=None, tree_tokens=None, target_tokens=None,
                        target_logits=None, max_path=16, k_tree=None, v_tree=None, k_cache=None, v_cache=None,
                        page_table=None, kv_len=None, kv_len_out=None, accept_path=None, req_range=None,
                        n_tree_rows=None, workspace=None):
    """CPU stand-in for the two record kernels of as_accept_tokens (test
    infrastructure: the oracle's walk and commit, same arguments and record
    layout as the library call), injected into dist.accept_and_commit."""
    to = tree_offsets.numpy()
    n = len(to) - 1
    rec = accept_path
    if phase == 3:  # AS_ACCEPT_WALK_RECORDS: rows [b, e) of this rank's requests
        b, e = req_range
        if e > b:
            sub_to = (to[b:e + 1] - to[b]).astype(np.int32)
            rows = slice(int(to[b]), int(to[e]))
            r = oracle.accept_walk(sub_to, tree_parent.numpy()[rows], tree_tokens.numpy()[rows],
                                   target_tokens=target_tokens.numpy()[rows], max_path=max_path)
            rec[b:e, 0] = torch.from_numpy(r["accept_len"])
            rec[b:e, 1] = torch.from_numpy(r["bonus_token"])
            rec[b:e, 2:] = torch.from_numpy(r["accept_path"])
    elif phase == 4:  # AS_ACCEPT_COMMIT_RECORDS: every request, this rank's heads
        kc, vc, kl = k_cache.numpy(), v_cache.numpy(), kv_len.numpy().copy()
        oracle.commit(to, rec[:n, 0].numpy().copy(), rec[:n, 2:].numpy().copy(), k_tree.numpy(), v_tree.numpy(),
                      kc, vc, page_table.numpy(), kl)
        (kv_len_out if kv_len_out is not None else kv_len).copy_(torch.from_numpy(kl))
    else:
        raise AssertionError(phase)


def _worker_library(rank, world, port, q):
    """dist.accept_and_commit / ShardedAccept -- the library's multi-GPU call --
    over gloo with the CPU record kernels: two batches of different sizes
    through one ShardedAccept (the record buffer is re-sized when ceil(n/world)
    changes), each equal to the single-process walk + commit of this rank's heads."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sharded = ShardedAccept(accept_fn=_cpu_record_kernels)
    ok = True
    for n, seed in ((9, 21), (30, 22), (3, 23), (30, 24)):
        to, par, toks, tgt = _walk_inputs(seed, n)
        mpth = 20
        rng = np.random.default_rng(seed)
        R = int(to[-1])
        n_kv, d, ps = 2 * world, 8, 4
        kv_len = rng.integers(0, 9, n).astype(np.int32)
        table, n_pages = synth.paged_kv(rng, kv_len, ps, extra_slots=mpth + 2)
        kt = rng.standard_normal((R, n_kv, d)).astype(np.float32)
        vt = rng.standard_normal((R, n_kv, d)).astype(np.float32)
        kc = rng.standard_normal((n_pages, n_kv, ps, d)).astype(np.float32)
        vc = rng.standard_normal((n_pages, n_kv, ps, d)).astype(np.float32)
        full = oracle.accept_walk(to, par, toks, target_tokens=tgt, max_path=mpth)
        kc_all, vc_all, kl_all = kc.copy(), vc.copy(), kv_len.copy()
        oracle.commit(to, full["accept_len"], full["accept_path"], kt, vt, kc_all, vc_all, table, kl_all)
        h0, h1 = head_range(n_kv, rank, world)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        kc_me, vc_me = T(kc[:, h0:h1]), T(vc[:, h0:h1])
        kl_in, kl_out = T(kv_len), torch.full((n,), -1, dtype=torch.int32)
        rec = sharded(T(to), T(par), T(toks), T(kt[:, h0:h1]), T(vt[:, h0:h1]), kc_me, vc_me, T(table), kl_in,
                      max_path=mpth, target_tokens=T(tgt), kv_len_out=kl_out)
        s = (n + world - 1) // world
        ok = ok and tuple(rec.shape) == (world * s, 2 + mpth)
        ok = ok and np.array_equal(rec[:n, 0].numpy(), full["accept_len"])
        ok = ok and np.array_equal(rec[:n, 1].numpy(), full["bonus_token"])
        ok = ok and np.array_equal(rec[:n, 2:].numpy(), full["accept_path"])
        ok = ok and np.array_equal(kc_me.numpy(), kc_all[:, h0:h1]) and np.array_equal(vc_me.numpy(), vc_all[:, h0:h1])
        ok = ok and np.array_equal(kl_out.numpy(), kl_all) and np.array_equal(kl_in.numpy(), kv_len)
    # a mis-sized static buffer is refused, not silently misaligned
    to, par, toks, tgt = _walk_inputs(1, 5)
    try:
        accept_and_commit(None, torch.from_numpy(to), None, None, None, None, None, None, None, None, max_path=4,
                          records=torch.zeros((1, 6), dtype=torch.int32), accept_fn=_cpu_record_kernels)
        ok = False
    except ValueError:
        pass
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_library_accept_and_commit_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_library, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


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
