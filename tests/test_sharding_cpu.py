"""Unit sharding on CPU: bin packing, and the global fire
accounting over a world-size-2 gloo exchange against the oracle engine
(which is pinned to the reference's own runs, tests/test_oracle.py)."""

import os
import socket
from dataclasses import replace

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import hc_oracle as O
from paper_2601_13684_b200.engine import EngineConfig
from paper_2601_13684_b200.parallel import (LocalExchange, assign_units, merge_reports,
                                            order_fires, shard_units)
from paper_2601_13684_b200.reporting import RetrievalRecord, SimulationReport, StepRow
from paper_2601_13684_b200.workload import CONFIGS, plan_for

NL, L, T = 4, 64, 32
SHIFT = {0: 9, 1: 9, 2: 9, 3: 17}  # layers 0-2 drift together, layer 3 later


def _trace():
    """Dense HCTRACE1-style rows: per layer a pivot (head 0) and two satellites.
    Pivot rows put their mass on [0, 16) until the layer's shift, then on
    [32, 48) -- so several pivots fire at the same window boundary."""
    rng = np.random.default_rng(7)
    K = L + T
    H = 3
    idx = np.full((T + 1, NL, H, K), O.PAD_INDEX, dtype=np.uint32)
    sc = np.zeros((T + 1, NL, H, K), dtype=np.float32)
    for t in range(T + 1):
        n = L + t if t else L
        for l in range(NL):
            for h in range(H):
                row = rng.random(n).astype(np.float32) * 0.01
                hot = slice(32, 48) if t >= SHIFT[l] else slice(0, 16)
                if h == 0 or t == 0:
                    row[hot] += 1 + rng.random(16).astype(np.float32)
                idx[t, l, h, :n] = np.arange(n)
                sc[t, l, h, :n] = row
    roles = {(l, h): ("pivot" if h == 0 else "satellite") for l in range(NL) for h in range(H)}
    clusters = [((l, 0), ((l, 1), (l, 2))) for l in range(NL)]
    lengths = {(l, h): 10 + 3 * h for l in range(NL) for h in (1, 2)}
    return idx, sc, dict(prefill_len=L, bytes_per_kv_entry=512, roles=roles, clusters=clusters,
                         lengths=lengths, l_base_int=16, window=8, transfer_bandwidth=1000,
                         update_delay_steps=1, measure=False)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fires_by_step(events):
    out = {}
    for e in events:
        out.setdefault(e["trigger_step"], []).append(
            (0, tuple(e["pivot"]), int(e["transfer_bytes"])))
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_13684_b200.parallel import FireExchange

    idx, sc, kw = _trace()
    ref = O.replay(idx, sc, **kw)
    cfg = EngineConfig(transfer_bandwidth=kw["transfer_bandwidth"],
                       update_delay_steps=kw["update_delay_steps"])
    ex = FireExchange()
    cum = [0]
    got = {}
    for t, fires in sorted(_fires_by_step(ref["events"]).items()):
        mine = [f for f in fires if f[1][0] % world == rank]  # layers alternate between ranks
        for key, (done, _) in order_fires(t, ex.all_gather(mine), cum, cfg).items():
            got[(t, key[1])] = done
    q.put((rank, got, cum[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_trace_has_simultaneous_fires():
    idx, sc, kw = _trace()
    ref = O.replay(idx, sc, **kw)
    steps = [e["trigger_step"] for e in ref["events"]]
    assert len(ref["events"]) == 4 and steps.count(16) == 3 and steps.count(24) == 1
    # queued: the bandwidth model pushes later pivots' completions out
    assert len({e["completion_step"] for e in ref["events"] if e["trigger_step"] == 16}) == 3


def test_order_fires_two_ranks_matches_reference_accounting():
    idx, sc, kw = _trace()
    ref = O.replay(idx, sc, **kw)
    want = {(e["trigger_step"], tuple(e["pivot"])): e["completion_step"] for e in ref["events"]}
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got, cum in res:
        assert got == want  # every rank computes every completion step
        assert cum == sum(e["transfer_bytes"] for e in ref["events"])


def test_order_fires_local_equals_sequential():
    cfg = EngineConfig(transfer_bandwidth=1000, update_delay_steps=2)
    cum = [0, 500]
    fires = [(1, (3, 0), 700), (0, (2, 0), 1500), (0, (0, 0), 200)]
    out = order_fires(8, LocalExchange().all_gather(fires), cum, cfg)
    # sequence 0: pivots (0,0) then (2,0); sequence 1 separately
    assert out[(0, (0, 0))] == (10, 200) and out[(0, (2, 0))] == (10, 1700)
    assert out[(1, (3, 0))] == (10, 1200)
    assert cum == [1700, 1200]
    with pytest.raises(ValueError):
        order_fires(8, [[(0, (0, 0), 1)], [(0, (0, 0), 1)]], [0], cfg)


@pytest.mark.parametrize("name,world", [("cfg3", 2), ("cfg3", 8), ("cfg5", 8), ("cfg2", 4)])
def test_assign_units_covers_and_balances(name, world):
    w = CONFIGS[name]
    tax, plan = plan_for(w)
    owned = assign_units(tax, plan, w.batch, world, w.decode_steps)
    assert owned.shape == (world, w.batch, w.num_layers, tax.heads_per_layer)
    assert (owned.sum(axis=0) == 1).all()  # every unit on exactly one rank
    for c in tax.clusters:  # clusters never split
        for r in range(world):
            for s in c.satellites:
                assert (owned[r, :, c.pivot[0], c.pivot[1]] == owned[r, :, s[0], s[1]]).all()
    units = shard_units(tax, plan, w.batch, w.decode_steps)
    load = np.zeros(world)
    for b, _, members, wt in units:
        r = int(np.flatnonzero(owned[:, b, members[0][0], members[0][1]])[0])
        load[r] += wt
    heaviest = max(u[3] for u in units)
    assert load.max() - load.min() <= heaviest  # LPT bound


def test_merge_reports_sums_partials_and_unions_events():
    def rep(rows, events):
        return SimulationReport(policy="heterocache", trace_sha256="", num_layers=2,
                                heads_per_layer=2, prefill_len=8, decode_steps=1,
                                budget_ceiling=1.0, update_delay_steps=1, rows=tuple(rows),
                                events=tuple(events))

    row = StepRow(step=1, recall=float("nan"), gpu_entries=10, extra_entries=3,
                  bytes_in_flight=5, cumulative_bytes=9, retrieval_flag=1)
    e0 = RetrievalRecord(trigger_step=1, pivot=(1, 0), completion_step=2, transfer_bytes=4,
                         fetches=())
    e1 = RetrievalRecord(trigger_step=1, pivot=(0, 0), completion_step=2, transfer_bytes=5,
                         fetches=())
    m = merge_reports([rep([row], [e0]), rep([replace(row, gpu_entries=7, extra_entries=1)], [e1])])
    assert m.rows[0].gpu_entries == 17 and m.rows[0].extra_entries == 4
    assert [e.pivot for e in m.events] == [(0, 0), (1, 0)]
    with pytest.raises(ValueError):
        merge_reports([rep([row], []), rep([replace(row, cumulative_bytes=1)], [])])


def test_combine_unit_outputs_takes_each_rank_rows():
    import torch

    from paper_2601_13684_b200.parallel import combine_unit_outputs

    B, NL, H, G, D = 2, 3, 4, 2, 5
    owned = np.zeros((2, B, NL, H), dtype=bool)
    owned[0, :, :, :2] = True
    owned[1, :, :, 2:] = True
    parts = [torch.full((B, NL, H * G, D), float(r)) for r in range(2)]
    out = combine_unit_outputs(parts, owned, G)
    assert (out[:, :, :2 * G] == 0).all() and (out[:, :, 2 * G:] == 1).all()
