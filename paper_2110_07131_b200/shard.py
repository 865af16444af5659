"""User sharding across ranks: the multi-GPU form of the hot path.

Reverse k-MIPS decides every user independently (Def. 2: u is in R_k(q)
iff q is in u's k-MIPS result over P u {q}), so one problem shards by users: each rank builds an
index over a contiguous range of user ids with the SAME items P and answers the same query batches;
only the per-query result lists are exchanged.  Contiguous id ranges keep the concatenation in rank
order ascending, so the gathered sets need no merge sort.  This is the paper's multicore scheme
(threads take disjoint blocks of users) across GPUs.

The exchange (gather_csr) is device-side: an all_gather of every rank's per-query counts, then an
all_gather of the rank's ids padded to the largest rank total, and a scatter of each rank's segments
into the global CSR -- all torch.distributed collectives on the ranks' tensors (NCCL over NVLink on
GPUs, gloo on CPU in the tests).  Per-rank work is the C ABI (rmips.py); this module only moves ids.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np


def user_shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, stop) of rank's users: contiguous, sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_csr(offsets, ids, start: int, group=None):
    """All ranks call this with their shard's CSR result (offsets [b + 1] int64, ids [total] int32 with
    shard-local user ids, torch tensors on the rank's device); every rank gets the global CSR result
    (offsets [b + 1] int64, ids [sum of totals] int32 global user ids, ascending per query)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = offsets.device
    b = offsets.numel() - 1
    counts = (offsets[1:] - offsets[:-1]).to(torch.int64)
    allc = [torch.empty_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts, group=group)
    C = torch.stack(allc)                                   # [world, b]
    totals = C.sum(1)                                       # [world]
    tmax = int(totals.max().item())
    pad = torch.zeros(max(tmax, 1), dtype=torch.int32, device=dev)
    pad[: ids.numel()] = ids.to(torch.int32) + int(start)  # global ids
    allp = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(allp, pad, group=group)
    per_q = C.sum(0)
    out_off = torch.zeros(b + 1, dtype=torch.int64, device=dev)
    out_off[1:] = torch.cumsum(per_q, 0)
    out_ids = torch.empty(int(out_off[-1].item()), dtype=torch.int32, device=dev)
    before = torch.cumsum(C, 0) - C                         # ids of lower ranks before rank r, per query
    qidx_all = torch.arange(b, device=dev)
    for r in range(world):
        t = int(totals[r].item())
        if t == 0:
            continue
        qidx = torch.repeat_interleave(qidx_all, C[r])     # query of each of rank r's ids
        loc_off = torch.cumsum(C[r], 0) - C[r]              # rank r's local offsets
        local = torch.arange(t, device=dev) - loc_off[qidx]
        dest = out_off[qidx] + before[r, qidx] + local
        out_ids[dest] = allp[r][:t]
    return out_off, out_ids


def merge_shards(parts: Sequence[Tuple[np.ndarray, np.ndarray]]) -> Tuple[np.ndarray, np.ndarray]:
    """Host reference of the merge: concatenate per-rank CSR results (global ids, rank order)."""
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
