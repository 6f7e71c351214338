"""Rank-range sharding of a trace store over GPUs.

One process per GPU. Shard p owns the records of ranks [lo_p, hi_p) (a
contiguous split of the layout's world), in their original store order, so
every per-rank prefix quantity of the analysis stays local. The engine
combines shards with NCCL collectives on its own stream (csrc/comm.cu); this
module is the host plumbing around it: the partition, and the NCCL
communicator bootstrap over torch.distributed (the unique id is broadcast
with the process group, gloo or nccl).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def shard_bounds(world_ranks: int, nshards: int) -> List[Tuple[int, int]]:
    """Contiguous rank ranges [lo, hi) covering [0, world_ranks); the last
    shard also owns any record rank >= world_ranks."""
    if nshards < 1:
        raise ValueError("nshards must be >= 1")
    out = []
    for p in range(nshards):
        lo = (world_ranks * p) // nshards
        hi = (world_ranks * (p + 1)) // nshards
        out.append((lo, hi if p + 1 < nshards else 0x7FFFFFFF))
    return out


def shard_of(rank: np.ndarray, world_ranks: int, nshards: int) -> np.ndarray:
    """Shard index of each record rank."""
    b = np.array([lo for lo, _ in shard_bounds(world_ranks, nshards)][1:], dtype=np.int64)
    return np.searchsorted(b, np.asarray(rank, dtype=np.int64), side="right")


def shard_records(records: np.ndarray, world_ranks: int, nshards: int,
                  shard: int) -> np.ndarray:
    """The shard's records, keeping store (emission) order."""
    return records[shard_of(records["rank"], world_ranks, nshards) == shard]


def init_engine_comm(ctx, group=None) -> None:
    """Create the engine's NCCL communicator across the torch.distributed
    group: rank 0 draws the unique id, the group broadcasts it."""
    import torch.distributed as dist

    from . import engine

    ws = dist.get_world_size(group)
    rk = dist.get_rank(group)
    if ws == 1:
        return
    obj = [engine.comm_unique_id() if rk == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(obj[0], ws, rk)
