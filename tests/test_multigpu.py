"""World-2 GPU test of the sharded path: two processes, one GPU each, NCCL; each rank
builds the CUDA index over its user shard and answers the same queries; shard.gather_csr exchanges the
per-query lists over NCCL; every rank's global sets equal the oracle's.  Skipped with fewer than two
GPUs (the graft GPU box has one: the plumbing is covered on CPU by test_multirank_cpu.py)."""
import os
import socket

import numpy as np
import pytest

import oracle
from synth import generator as gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if torch.cuda.device_count() < 2:
    pytest.skip("needs two GPUs", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, U, P, Qy, k, kmax, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        from paper_2110_07131_b200 import rmips
        from paper_2110_07131_b200.shard import gather_csr, user_shard
        dev = torch.device("cuda", rank)
        a, b = user_shard(U.shape[0], world, rank)
        idx = rmips.rmips_build_index(torch.from_numpy(U[a:b]).to(dev), torch.from_numpy(P).to(dev), kmax)
        off, ids = rmips.rmips_query(idx, torch.from_numpy(Qy).to(dev), k)
        g_off, g_ids = gather_csr(off, ids, a)
        np.savez(out_path + ".%d.npz" % rank, off=g_off.cpu().numpy(), ids=g_ids.cpu().numpy())
        idx.close()
    finally:
        dist.destroy_process_group()


def test_two_gpu_sharded_build_and_query(tmp_path):
    U, P = gen.random_instance(41, 5000, 800, 50, "skewed")
    Qy = np.concatenate([P[:40], gen.random_instance(42, 20, 1, 50, "skewed")[0]])
    out = str(tmp_path / "g")
    mp.spawn(_worker, args=(2, _free_port(), U, P, Qy, 7, 10, out), nprocs=2, join=True)
    sets = oracle.sets_from_member(oracle.rkmips_naive(U, P, Qy, 7))
    want_off = np.zeros(len(sets) + 1, np.int64)
    want_off[1:] = np.cumsum([len(s) for s in sets])
    want_ids = np.concatenate(sets)
    for r in range(2):
        got = np.load(out + ".%d.npz" % r)
        assert np.array_equal(got["off"], want_off) and np.array_equal(got["ids"], want_ids)
