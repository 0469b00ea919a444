"""Multi-GPU plumbing: sequence sharding and max-over-ranks timing.

HeteroCache units are independent across sequences: a pivot and its
satellites live in the same sequence and layer, and every sequence keeps its
own cumulative byte counter (engine.py:333-337), so sharding whole sequences
keeps completion steps exact with no data-path collective.  One process per
GPU (torchrun); NCCL for the timing reduction and the optional output gather,
gloo in the CPU tests.
"""

from __future__ import annotations


def shard_sequences(global_batch: int, world: int, rank: int) -> list:
    """Sequences owned by `rank` (round robin, every sequence exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, global_batch, world))


def max_over_ranks(values, device=None) -> list:
    """Element-wise max of per-rank timings (the bench's clock is the slowest rank)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(v) for v in values], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def gather_outputs(local):
    """All-gather per-shard attention outputs [b_local, ...] into rank order."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [local]
    parts = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local.contiguous())
    return parts
