"""User sharding across ranks: the multi-GPU form of the hot path.

Reverse k-MIPS decides every user independently (Def. 2: u is in R_k(q)
iff q is in u's k-MIPS result over P u {q}), so the users shard with no data-path collective:
each rank builds an index over a contiguous range of user ids with the SAME items, answers the
same query batch, and only the per-query result lists are gathered.  Contiguous id ranges keep
the concatenation in rank order ascending, so the gathered sets need no merge.

Host-side plumbing only (torch.distributed); the per-rank work is the C ABI (rmips.py).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def user_shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, stop) of rank's users: contiguous, sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def globalize(offsets: np.ndarray, ids: np.ndarray, start: int) -> Tuple[np.ndarray, np.ndarray]:
    """Shard-local CSR (user ids relative to the shard) -> global user ids."""
    return np.asarray(offsets, np.int64), np.asarray(ids, np.int64) + int(start)


def merge_shards(parts: Sequence[Tuple[np.ndarray, np.ndarray]]) -> Tuple[np.ndarray, np.ndarray]:
    """Concatenate per-rank CSR results (global ids, rank order) query by query."""
    nq = len(parts[0][0]) - 1
    counts = np.zeros(nq, np.int64)
    for off, _ in parts:
        if len(off) != nq + 1:
            raise ValueError("ranks answered different query batches")
        counts += np.diff(off)
    out_off = np.zeros(nq + 1, np.int64)
    np.cumsum(counts, out=out_off[1:])
    out_ids = np.empty(int(out_off[-1]), np.int64)
    cursor = out_off[:-1].copy()
    for off, ids in parts:
        for i in range(nq):
            a, b = off[i], off[i + 1]
            out_ids[cursor[i]:cursor[i] + (b - a)] = ids[a:b]
            cursor[i] += b - a
    return out_off, out_ids


def gather_sets(offsets: np.ndarray, ids: np.ndarray, start: int, group=None) -> Tuple[np.ndarray, np.ndarray]:
    """All ranks call this with their shard's CSR result; every rank gets the global CSR result
    (torch.distributed all_gather_object over `group`)."""
    import torch.distributed as dist

    mine = globalize(offsets, ids, start)
    world = dist.get_world_size(group)
    parts: List = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return merge_shards(parts)
