"""Multi-GPU glue: KV-head sharding of verification attention and the single
NCCL exchange of the hot path (BASELINE north_star).

* select is replicated (deterministic, bit-exact on every rank, no traffic);
* attention is sharded by KV head: rank p owns kv heads
  [p*n_kv/P, (p+1)*n_kv/P) and their G query heads (no collective);
* the acceptance walk is sharded by request (rank p walks requests
  [p*s, (p+1)*s), s = ceil(n/P)) and writes fixed-size int32 records
  {accept_len, bonus_token, path[max_path]} straight into its rows of a
  [P*s, 2 + max_path] buffer (as_accept_tokens AS_ACCEPT_WALK_RECORDS), ONE
  in-place all_gather_into_tensor over NCCL / NVLink fills the other ranks'
  rows, and every rank commits ALL requests' paths for ITS OWN kv heads from
  the records (AS_ACCEPT_COMMIT_RECORDS): 2 kernels + 1 collective, no packing.
Nothing else crosses NVLink: no KV, no activations, no logits.

`accept_and_commit(pg, ...)` is the library call (SURVEY §8(b) "Python
surface"); `ShardedAccept` keeps the record buffer static across calls (CUDA
graph capture) and re-sizes it whenever the request shard size changes.  The
record kernels are reached through `accept_fn` (default: the library's
`accept_tokens`), so the host protocol runs unchanged under gloo on CPU with a
stand-in (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(n_kv: int, rank: int, world: int):
    """KV heads owned by `rank` (n_kv must be divisible by world)."""
    if n_kv % world:
        raise ValueError(f"n_kv={n_kv} not divisible by world={world}")
    per = n_kv // world
    return rank * per, (rank + 1) * per


def request_range(n: int, rank: int, world: int):
    """Requests walked by `rank`: [b, e) with shard size s = ceil(n/world)."""
    s = (n + world - 1) // world
    b = min(n, rank * s)
    return b, min(n, b + s), s


def pack_records(accept_len, accept_path, bonus_token, b, e, s):
    """Rows [b, e) of the walk outputs -> an int32 [s, 2 + max_path] record block
    (rows past e are padding, accept_len = 0)."""
    mp = accept_path.shape[1]
    rec = torch.zeros((s, 2 + mp), dtype=torch.int32, device=accept_len.device)
    k = e - b
    if k > 0:
        rec[:k, 0] = accept_len[b:e]
        rec[:k, 1] = bonus_token[b:e]
        rec[:k, 2:] = accept_path[b:e]
    return rec


def unpack_records(gathered, n, accept_len, accept_path, bonus_token):
    """[world*s, 2+mp] gathered records -> the first n rows of the outputs (in place)."""
    accept_len.copy_(gathered[:n, 0])
    bonus_token.copy_(gathered[:n, 1])
    accept_path.copy_(gathered[:n, 2:])


def all_gather_records(rec, world, group=None):
    out = torch.empty((world * rec.shape[0], rec.shape[1]), dtype=rec.dtype, device=rec.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    return out


def record_shard(records, rank, s):
    """This rank's rows of the [world*s, 2+mp] record buffer (a contiguous view)."""
    return records[rank * s:(rank + 1) * s]


def all_gather_in_place(records, rank, world, group=None, s=None):
    """Fill every rank's rows of `records` from the owner rank (in place).  The
    shard size `s` defaults to the buffer's rows / world; pass it explicitly
    when the buffer may be larger than world * ceil(n / world)."""
    if s is None:
        s = records.shape[0] // world
    view = records[:world * s]
    dist.all_gather_into_tensor(view, record_shard(records, rank, s), group=group)
    return records


def record_buffer(n: int, world: int, max_path: int, device) -> torch.Tensor:
    """The [world * ceil(n/world), 2 + max_path] int32 record buffer of one step."""
    s = (n + world - 1) // world
    return torch.zeros((max(world * s, 1), 2 + max_path), dtype=torch.int32, device=device)


def accept_and_commit(pg, tree_offsets, tree_parent, tree_tokens, k_tree, v_tree, k_cache, v_cache, page_table,
                      kv_len, *, max_path, target_tokens=None, target_logits=None, kv_len_out=None, records=None,
                      n_tree_rows=None, workspace=None, accept_fn=None):
    """One multi-GPU acceptance step: this rank walks its
    request shard into its rows of `records` (WALK_RECORDS), one in-place
    all_gather_into_tensor on `pg` completes the records on every rank, and
    every rank commits every request's accepted path into ITS kv-head shard of
    the paged cache (COMMIT_RECORDS; `k_tree/v_tree/k_cache/v_cache` are this
    rank's head slices; kv_len += accept_len, out of place into kv_len_out when
    given).  Returns the [world*s, 2 + max_path] records {len, bonus, path}.

    `records` (optional) must have exactly world * ceil(n / world) rows (a
    static buffer for graph capture; see ShardedAccept).  `accept_fn` defaults
    to the library's accept_tokens (the CUDA record kernels)."""
    if accept_fn is None:
        from . import accept_tokens as accept_fn
        from . import AS_ACCEPT_COMMIT_RECORDS, AS_ACCEPT_WALK_RECORDS
    else:
        AS_ACCEPT_WALK_RECORDS, AS_ACCEPT_COMMIT_RECORDS = 3, 4
    world = dist.get_world_size(pg)
    rank = dist.get_rank(pg)
    n = tree_offsets.numel() - 1
    b, e, s = request_range(n, rank, world)
    if records is None:
        records = record_buffer(n, world, max_path, tree_offsets.device)
    if records.shape != (max(world * s, 1), 2 + max_path) or records.dtype != torch.int32:
        raise ValueError(f"records must be int32 [{world * s}, {2 + max_path}] for n={n}, world={world}; "
                         f"got {tuple(records.shape)} {records.dtype}")
    common = dict(max_path=max_path, k_tree=k_tree, v_tree=v_tree, k_cache=k_cache, v_cache=v_cache,
                  page_table=page_table, kv_len=kv_len, kv_len_out=kv_len_out, accept_path=records,
                  n_tree_rows=n_tree_rows, workspace=workspace)
    accept_fn(AS_ACCEPT_WALK_RECORDS, tree_offsets, tree_parent, tree_tokens, target_tokens=target_tokens,
              target_logits=target_logits, req_range=(b, e), **common)
    if world > 1:
        all_gather_in_place(records, rank, world, group=pg, s=s)
    accept_fn(AS_ACCEPT_COMMIT_RECORDS, tree_offsets, tree_parent, tree_tokens, **common)
    return records


class ShardedAccept:
    """accept_and_commit with a static record buffer (captured into CUDA graphs),
    re-allocated whenever ceil(n / world) or max_path changes."""

    def __init__(self, pg=None, accept_fn=None):
        self.pg = pg
        self.accept_fn = accept_fn
        self.records = None

    def __call__(self, tree_offsets, tree_parent, tree_tokens, k_tree, v_tree, k_cache, v_cache, page_table, kv_len,
                 *, max_path, **kw):
        world = dist.get_world_size(self.pg)
        n = tree_offsets.numel() - 1
        s = (n + world - 1) // world
        want = (max(world * s, 1), 2 + max_path)
        if self.records is None or tuple(self.records.shape) != want:
            self.records = record_buffer(n, world, max_path, tree_offsets.device)
        return accept_and_commit(self.pg, tree_offsets, tree_parent, tree_tokens, k_tree, v_tree, k_cache, v_cache,
                                 page_table, kv_len, max_path=max_path, records=self.records,
                                 accept_fn=self.accept_fn, **kw)
