"""N > 1 path on CPU (world_size 2 and 3, gloo): user sharding and the device-side CSR gather
(shard.gather_csr: all_gather of counts, padded all_gather of ids, scatter into the global CSR) give
the single-process answer.  The per-rank reverse k-MIPS here is the oracle (this is the host-side
plumbing test; tests/test_multigpu.py runs the same gather over NCCL with the CUDA path per rank when
two GPUs are present)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2110_07131_b200.shard import gather_csr, merge_shards, user_shard
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
        g_off, g_ids = gather_csr(torch.from_numpy(off), torch.from_numpy(ids.astype(np.int32)), a)
        np.savez(out_path + ".%d.npz" % rank, off=g_off.numpy(), ids=g_ids.numpy())
        # the timing reduction bench.py uses (max over ranks)
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
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_gather_csr_equals_single_process(tmp_path, world):
    U, P = gen.random_instance(31, 301, 90, 12, "skewed")
    Qy = np.concatenate([P[:10], gen.random_instance(32, 6, 1, 12, "skewed")[0]])
    k = 5
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(world, _free_port(), U, P, Qy, k, out), nprocs=world, join=True)
    want_off, want_ids = _csr(oracle.rkmips_naive(U, P, Qy, k))
    for r in range(world):  # every rank holds the global result
        got = np.load(out + ".%d.npz" % r)
        assert np.array_equal(got["off"], want_off)
        assert np.array_equal(got["ids"], want_ids)
