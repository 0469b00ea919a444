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


def _fire_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_13684_b200.parallel import TensorFireExchange

    ex = TensorFireExchange(capacity=3)
    got = []
    # boundary 1: both ranks fire; boundary 2: only rank 1; boundary 3: nobody
    mine = [[(0, (rank, 0), 1000 + rank), (1, (rank + 2, 0), 7)], [(1, (5, 0), 42)] if rank else [],
            []]
    for fires in mine:
        got.append(ex.all_gather(fires))
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_tensor_fire_exchange_gathers_every_ranks_fires():
    """parallel.TensorFireExchange (the bench's fixed-size fire all-gather) returns
    every rank's (sequence, pivot, bytes) fires in rank order, on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fire_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [[[(0, (0, 0), 1000), (1, (2, 0), 7)], [(0, (1, 0), 1001), (1, (3, 0), 7)]],
            [[], [(1, (5, 0), 42)]], [[], []]]
    assert res[0] == res[1] == want


def test_slab_units_partition():
    import numpy as np

    from paper_2601_13684_b200.parallel import slab_units
    from paper_2601_13684_b200.workload import LLAMA3_8B, roles_for

    tax = roles_for(LLAMA3_8B, 4)
    own = slab_units(tax, 2, 4)  # 8 (sequence, layer) pairs over 4 ranks
    assert own.shape == (4, 2, 4, 8) and (own.sum(0) == 1).all()
    for r in range(4):  # rank r: pairs 2r, 2r+1 -> one contiguous slab of O
        flat = own[r].reshape(8, 8).any(1)
        assert np.flatnonzero(flat).tolist() == [2 * r, 2 * r + 1]
    with pytest.raises(ValueError):
        slab_units(tax, 1, 3)
