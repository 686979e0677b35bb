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

The packing helpers are plain torch ops (device-agnostic) so the protocol is
tested with the gloo backend on CPU (tests/test_dist_gloo.py).
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
    """Requests walked by `rank`: [b, e) with shard size ceil(n/world)."""
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


def all_gather_in_place(records, rank, world, group=None):
    """Fill every rank's rows of `records` from the owner rank (in place)."""
    s = records.shape[0] // world
    dist.all_gather_into_tensor(records, record_shard(records, rank, s), group=group)
    return records


class ShardedAccept:
    """WALK_RECORDS on this rank's request shard -> in-place all-gather ->
    COMMIT_RECORDS (every rank, its own kv heads)."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.records = None

    def accept_and_commit(self, W):
        import paper_2501_12162_b200 as ada
        from bench import run_accept_records  # the bench's call wrapper (same arguments)
        n = W["n"]
        b, e, s = request_range(n, self.rank, self.world)
        if self.records is None:
            self.records = torch.zeros((self.world * s, 2 + W["max_path"]), dtype=torch.int32,
                                       device=W["kv_len"].device)
        run_accept_records(W, ada.AS_ACCEPT_WALK_RECORDS, self.records, req_range=(b, e))
        all_gather_in_place(self.records, self.rank, self.world, self.group)
        run_accept_records(W, ada.AS_ACCEPT_COMMIT_RECORDS, self.records)
