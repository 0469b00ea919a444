"""World-size-2 gloo tests of the multi-GPU plumbing (CPU only)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_13684_b200.parallel import gather_outputs, max_over_ranks, shard_sequences

    mine = shard_sequences(8, world, rank)
    times = max_over_ranks([10.0 + rank, 5.0 - rank])
    local = torch.full((len(mine), 3), float(rank))
    parts = gather_outputs(local)
    q.put((rank, mine, times, [p.tolist() for p in parts]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_reduction():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = sorted(s for _, mine, _, _ in res for s in mine)
    assert owned == list(range(8))  # every sequence exactly once
    for _, _, times, parts in res:
        assert times == [11.0, 5.0]  # max over ranks, element-wise
        assert parts[0] == [[0.0] * 3] * 4 and parts[1] == [[1.0] * 3] * 4


def test_shard_validation():
    from paper_2601_13684_b200.parallel import shard_sequences

    assert shard_sequences(5, 2, 1) == [1, 3]
    with pytest.raises(ValueError):
        shard_sequences(4, 2, 2)
