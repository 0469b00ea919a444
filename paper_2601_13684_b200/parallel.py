"""Multi-GPU plumbing.

Two partitionings, one process per GPU (torchrun):

* **sequence shards** (``shard_sequences``): HeteroCache units are independent
  across sequences -- a pivot and its satellites live in the same sequence and
  layer, and every sequence keeps its own cumulative byte counter
  (engine.py:333-337) -- so whole sequences per rank need no data-path
  collective at all (the bench's default, weak scaling).
* **unit shards** (``assign_units``): one sequence's (layer, cluster-or-loner
  head) units spread over ranks, greedily bin-packed by per-step bytes.  The
  only cross-rank dependency is the byte accounting: a fire's completion step
  is ``max(t + delay, ceil(cumulative_bytes / bandwidth))`` over ONE running
  counter per sequence, accumulated in sorted pivot order (engine.py:313,
  333-337).  At every window boundary each rank contributes its fires (a few
  bytes per firing pivot) through ``FireExchange``; ``order_fires`` then
  replays the reference's accumulation over the union on every rank, so
  completion steps -- and hence which steps see stale satellites -- are
  exactly the reference's.  ``merge_reports`` sums the per-rank partial
  StepRows and unions the events.

* **slabs** (``slab_units``, the bench's N>1 default): rank r owns the
  contiguous range [r*S, (r+1)*S) of the batch's (sequence, layer) pairs,
  S = B*NL / world -- the north star's (batch, KV-head) split of ONE batch
  (strong scaling).  Clusters are layer-local, so no cluster splits; each
  rank's query / output rows are one contiguous slab of O[B, NL, Hq, d], so
  the per-step output all-gather lands straight in place
  (``all_gather_into_tensor``, no index shuffle).  A sequence whose layers
  straddle two ranks shares its byte counter through the fire exchange.

``TensorFireExchange`` is the fire exchange as one fixed-size tensor
all-gather (NCCL on a side stream, so it runs beside the step's attention;
gloo on host tensors for the single-GPU functional tests).
"""

from __future__ import annotations

from math import ceil

import numpy as np


def shard_sequences(global_batch: int, world: int, rank: int) -> list:
    """Sequences owned by `rank` (round robin, every sequence exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, global_batch, world))


def shard_units(taxonomy, plan, batch: int, max_decode: int, *, sink_count: int = 4,
                recency_window: int = 8):
    """The indivisible shard units of a batch: (sequence, layer, members, bytes/step).

    A cluster (pivot + satellites) is one unit -- satellites are refilled from
    the pivot's row (engine.py:326-329) -- every other head is its own unit.
    The weight is the unit's resident rows at mid-decode, i.e. its K4 bytes.
    """
    L = plan.prefill_len
    units = []
    in_cluster = {}
    for c in taxonomy.clusters:
        for m in (c.pivot, *c.satellites):
            in_cluster[tuple(m)] = c
    full = set(taxonomy.full_heads())

    def rows(hd):
        if hd in full:
            return L + max_decode // 2
        k = min(plan.lengths.get(hd, 0), L)
        return k + min(sink_count, L) + recency_window + max_decode // 2

    seen = set()
    for b in range(batch):
        for l in range(taxonomy.num_layers):
            for h in range(taxonomy.heads_per_layer):
                hd = (l, h)
                if (b, hd) in seen:
                    continue
                c = in_cluster.get(hd)
                members = tuple(sorted((tuple(c.pivot), *map(tuple, c.satellites)))) if c else (hd,)
                for m in members:
                    seen.add((b, m))
                units.append((b, l, members, sum(rows(m) for m in members)))
    return units


def assign_units(taxonomy, plan, batch: int, world: int, max_decode: int, **kw) -> np.ndarray:
    """owned[rank][b, layer, head] (bool): longest-processing-time greedy bin
    packing of ``shard_units`` (heaviest first, to the least-loaded rank, ties
    to the lower rank): deterministic, every unit on exactly one rank."""
    if world < 1:
        raise ValueError(f"bad world {world}")
    units = shard_units(taxonomy, plan, batch, max_decode, **kw)
    order = sorted(range(len(units)), key=lambda i: (-units[i][3], i))
    load = [0] * world
    owned = np.zeros((world, batch, taxonomy.num_layers, taxonomy.heads_per_layer), dtype=bool)
    for i in order:
        b, _, members, w = units[i]
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += w
        for (l, h) in members:
            owned[r, b, l, h] = True
    return owned


def slab_units(taxonomy, batch: int, world: int) -> np.ndarray:
    """owned[rank][b, layer, head]: rank r owns (sequence, layer) pairs
    [r*S, (r+1)*S) in (b, layer) order, S = batch*num_layers / world."""
    NL, H = taxonomy.num_layers, taxonomy.heads_per_layer
    n = batch * NL
    if world < 1 or n % world:
        raise ValueError(f"{batch} x {NL} (sequence, layer) pairs do not split over {world} ranks")
    S = n // world
    owned = np.zeros((world, n, H), dtype=bool)
    for r in range(world):
        owned[r, r * S:(r + 1) * S] = True
    return owned.reshape(world, batch, NL, H)


def order_fires(step: int, gathered, cumulative: list, cfg) -> dict:
    """Completion steps of one boundary's fires over all ranks.

    gathered: per-rank lists of (sequence, pivot, transfer_bytes).  Per
    sequence the fires are taken in sorted pivot order -- the order the
    reference's decode_step visits pivots (engine.py:313, taxonomy.pivots() is
    sorted) -- and each adds its bytes to that sequence's one running counter
    before its completion step is computed (engine.py:333-337).  `cumulative`
    (per sequence) is updated in place; returns {(sequence, pivot): (completion,
    cumulative_bytes_after)}.
    """
    fires = sorted((int(b), tuple(p), int(n)) for part in gathered for (b, p, n) in part)
    out = {}
    for b, p, n in fires:
        if (b, p) in out:
            raise ValueError(f"pivot {p} of sequence {b} fired on two ranks")
        cumulative[b] += n
        done = max(step + cfg.update_delay_steps, ceil(cumulative[b] / cfg.transfer_bandwidth))
        out[(b, p)] = (done, cumulative[b])
    return out


class LocalExchange:
    """Single-process exchange (no other ranks)."""

    world = 1
    rank = 0

    def all_gather(self, obj) -> list:
        return [obj]


class FireExchange:
    """all_gather of small host objects over a torch.distributed group (gloo:
    the payload is a few bytes per firing pivot, host-side)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, obj) -> list:
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out


class TensorFireExchange:
    """The boundary fire exchange as ONE fixed-size all-gather of a tensor.

    Each rank packs its fires (sequence, pivot layer, pivot head, bytes) into a
    [capacity + 1, 4] int64 block (row 0: the count) and all-gathers the blocks
    of every rank.  With NCCL the gather runs on a side stream, so it does not
    wait for (and runs beside) the attention already queued on the decode
    stream; the host then reads back only that side stream.  gloo (functional
    tests on one GPU) gathers host tensors.
    """

    def __init__(self, capacity: int, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cap = max(1, int(capacity))
        self.nccl = dist.get_backend(group) == "nccl"
        dev = "cuda" if self.nccl else "cpu"
        self.send = torch.zeros(self.cap + 1, 4, dtype=torch.int64, device=dev)
        self.recv = torch.zeros(self.world, self.cap + 1, 4, dtype=torch.int64, device=dev)
        self.stage = torch.zeros(self.cap + 1, 4, dtype=torch.int64,
                                 pin_memory=self.nccl)
        self.stream = torch.cuda.Stream() if self.nccl else None

    def all_gather(self, obj) -> list:
        import torch
        import torch.distributed as dist

        if len(obj) > self.cap:
            raise ValueError(f"{len(obj)} fires exceed the exchange capacity {self.cap}")
        st = self.stage
        st[0, 0] = len(obj)
        for i, (b, p, n) in enumerate(obj):
            st[i + 1, 0], st[i + 1, 1], st[i + 1, 2], st[i + 1, 3] = int(b), p[0], p[1], int(n)
        if self.nccl:
            with torch.cuda.stream(self.stream):
                self.send.copy_(st, non_blocking=True)
                dist.all_gather_into_tensor(self.recv.view(-1, 4), self.send, group=self.group)
                host = self.recv.cpu()  # waits on this side stream only
        else:
            self.send.copy_(st)
            dist.all_gather_into_tensor(self.recv.view(-1, 4), self.send, group=self.group)
            host = self.recv
        out = []
        for r in range(self.world):
            n = int(host[r, 0, 0])
            out.append([(int(x[0]), (int(x[1]), int(x[2])), int(x[3]))
                        for x in host[r, 1:n + 1].tolist()])
        return out


def merge_reports(parts):
    """One sequence's SimulationReport from the per-rank partial reports of a
    unit-sharded run: gpu_entries / extra_entries are sums over heads
    (engine.py:276-288), so the partials add; bytes_in_flight, cumulative_bytes
    and retrieval_flag are already global on every rank (order_fires); events
    are the union in (trigger_step, pivot) order, the order decode_step emits
    them."""
    from dataclasses import replace

    base = parts[0]
    if len({len(p.rows) for p in parts}) != 1:
        raise ValueError("ranks report different numbers of steps")
    rows = []
    for rs in zip(*(p.rows for p in parts)):
        r0 = rs[0]
        for r in rs[1:]:
            if (r.step, r.bytes_in_flight, r.cumulative_bytes, r.retrieval_flag) != \
                    (r0.step, r0.bytes_in_flight, r0.cumulative_bytes, r0.retrieval_flag):
                raise ValueError(f"ranks disagree on the global fields of step {r0.step}")
        extra = -1 if any(r.extra_entries < 0 for r in rs) else sum(r.extra_entries for r in rs)
        rows.append(replace(r0, gpu_entries=sum(r.gpu_entries for r in rs), extra_entries=extra))
    events = sorted((e for p in parts for e in p.events), key=lambda e: (e.trigger_step, e.pivot))
    return replace(base, rows=tuple(rows), events=tuple(events))


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


def combine_unit_outputs(parts, owned, group: int):
    """Assemble O[B, NL, H*G, D] from per-rank outputs of a unit-sharded step:
    rank r holds the query rows of its owned (b, layer, kv_head) units."""
    import torch

    out = parts[0].clone()
    own = torch.as_tensor(owned)  # [world, B, NL, H]
    for r in range(1, len(parts)):
        m = own[r].to(out.device).repeat_interleave(group, dim=2)  # [B, NL, H*G]
        out[m] = parts[r][m]
    return out
