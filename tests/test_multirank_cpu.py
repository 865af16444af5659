"""N > 1 path on CPU (world_size 2, gloo): user sharding and the gathered result sets equal the
single-process answer.  The per-rank reverse k-MIPS here is the oracle (this is the host-side
plumbing test; the GPU path per rank is the same C ABI the parity tests cover)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2110_07131_b200.shard import gather_sets, merge_shards, user_shard
from synth import generator as gen


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _csr(member):
    sets = oracle.sets_from_member(member)
    off = np.zeros(len(sets) + 1, np.int64)
    off[1:] = np.cumsum([len(x) for x in sets])
    ids = np.concatenate(sets).astype(np.int64) if off[-1] else np.zeros(0, np.int64)
    return off, ids


def _worker(rank, world, port, U, P, Qy, k, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = user_shard(U.shape[0], world, rank)
        off, ids = _csr(oracle.rkmips_naive(U[a:b], P, Qy, k))  # shard-local user ids
        g_off, g_ids = gather_sets(off, ids, a)
        if rank == 0:
            np.savez(out_path, off=g_off, ids=g_ids)
        # the timing reduction bench.py uses (max over ranks)
        import torch
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
    finally:
        dist.destroy_process_group()


def test_user_shard_partitions():
    for n in (0, 1, 7, 128, 1001):
        for world in (1, 2, 3, 8):
            spans = [user_shard(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_merge_shards_keeps_ascending_order():
    p0 = (np.array([0, 2, 2]), np.array([1, 4]))
    p1 = (np.array([0, 1, 3]), np.array([7, 5, 9]))
    off, ids = merge_shards([p0, p1])
    assert off.tolist() == [0, 3, 5] and ids.tolist() == [1, 4, 7, 5, 9]


@pytest.mark.timeout(300)
def test_two_rank_gloo_gather_equals_single_process(tmp_path):
    U, P = gen.random_instance(31, 301, 90, 12, "skewed")
    Qy = np.concatenate([P[:10], gen.random_instance(32, 6, 1, 12, "skewed")[0]])
    k = 5
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, _free_port(), U, P, Qy, k, out), nprocs=2, join=True)
    got = np.load(out)
    want_off, want_ids = _csr(oracle.rkmips_naive(U, P, Qy, k))
    assert np.array_equal(got["off"], want_off)
    assert np.array_equal(got["ids"], want_ids)
