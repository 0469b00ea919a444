"""Unit-sharded decoding on one B200: two or three ranks
(processes on cuda:0, gloo fire exchange -- host data only, no kernel waits
on another rank) each hold a share of the (sequence, layer, cluster-or-loner)
units, in boundary mode and in sliding mode (eval_every_step) with delay 3.  The
merged reports must equal the unsharded decoder's (which tests/
test_decoder_gpu.py pins to the oracle engine), event for event and row for
row, with a bandwidth-limited link so that completion steps depend on the
reference's global accumulation order across ranks; the combined outputs
must be bit-identical (every unit runs the same tiles and combine)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

B, NL, L, T, SHIFT = 2, 4, 700, 40, 13
BANDWIDTH = 12000  # bytes per step: simultaneous fires queue behind each other


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {  # name: (world, EngineConfig overrides)
    "boundary_w2": (2, dict(window=8, update_delay_steps=1)),
    "sliding_delay3_w3": (3, dict(window=6, update_delay_steps=3, eval_every_step=True)),
}


def _run(owned=None, exchange=None, cfg_kw=None):
    import torch

    from paper_2601_13684_b200.decoder import HeteroCacheDecoder
    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.workload import ModelShape, SyntheticKV, Workload, plan_for

    model = ModelShape("tiny", NL, 32, 8)  # Llama role mix: pivot, 4 satellites, 2 anchors, volatile
    tax, plan = plan_for(Workload("tiny", model, L, B, 0.10, T, 0, layers=NL))
    cfg = EngineConfig(transfer_bandwidth=BANDWIDTH, **(cfg_kw or CASES["boundary_w2"][1]))
    dec = HeteroCacheDecoder(tax, plan, cfg, batch=B, group=model.group, max_decode=T, chunk=256,
                             owned=owned, exchange=exchange)
    gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=plan.l_base_int, seed=5)
    for l in range(NL):
        k, v, q = gen.layer_kv(l)
        dec.prefill_layer(l, k, v, q)
    torch.cuda.synchronize()
    dec.finish_prefill()
    outs = []
    for t in range(1, T + 1):
        q, kn, vn = gen.step_inputs(t, SHIFT)
        o = torch.zeros_like(q)
        dec.decode_step(t, q, kn, vn, o)
        outs.append(o)
    reports = [dec.report(b, T) for b in range(B)]
    o = torch.stack(outs).cpu()
    dec.close()
    return tax, plan, reports, o


def _worker(rank, world, port, q, case):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_13684_b200.parallel import FireExchange, assign_units
        from paper_2601_13684_b200.workload import ModelShape, Workload, plan_for

        model = ModelShape("tiny", NL, 32, 8)
        tax, plan = plan_for(Workload("tiny", model, L, B, 0.10, T, 0, layers=NL))
        owned = assign_units(tax, plan, B, world, T)
        _, _, reports, o = _run(owned[rank], FireExchange(), CASES[case][1])
        q.put((rank, owned, reports, o.float().numpy()))
    except Exception as e:  # surface the failure instead of hanging the parent
        q.put((rank, None, repr(e), None))
        raise
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_unit_sharding_matches_unsharded(case):
    from paper_2601_13684_b200.parallel import merge_reports

    world, cfg_kw = CASES[case]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[1] is not None, f"rank {r[0]} failed: {r[2]}"
    owned = res[0][1]
    assert (owned.sum(axis=0) == 1).all() and all(owned[r].any() for r in range(world))

    tax, plan, ref_reports, ref_o = _run(cfg_kw=cfg_kw)
    fired, firing_ranks = 0, set()
    for b in range(B):
        merged = merge_reports([res[r][2][b] for r in range(world)])
        assert merged.events == ref_reports[b].events, f"sequence {b}: events differ"
        assert len(merged.rows) == len(ref_reports[b].rows) == T + 1
        for m, e in zip(merged.rows, ref_reports[b].rows):  # recall is NaN (no measure mode)
            assert (m.step, m.gpu_entries, m.extra_entries, m.bytes_in_flight, m.cumulative_bytes,
                    m.retrieval_flag) == (e.step, e.gpu_entries, e.extra_entries,
                                          e.bytes_in_flight, e.cumulative_bytes, e.retrieval_flag)
        firing_ranks |= {int(np.flatnonzero(owned[:, b, e.pivot[0], e.pivot[1]])[0])
                         for e in merged.events}
        fired += len(merged.events)
        completions = [e.completion_step for e in merged.events]
        assert len(set(completions)) > 1  # the link model queued them
    assert fired >= 2 * B and len(firing_ranks) >= 2  # several pivots fired, on several ranks
    # combined outputs: rank r's rows of the query heads of its units
    ref = ref_o.float().numpy()
    G = 4
    comb = res[0][3].copy()
    for r in range(1, world):
        m = np.repeat(owned[r], G, axis=2)  # [B, NL, H*G]
        comb[:, m] = res[r][3][:, m]
    assert np.array_equal(comb, ref)


def test_sharded_engine_refuses_measure_mode_and_split_clusters():
    """Measure mode needs every head of every sequence; a satellite must live
    with its pivot (hc_engine_create_sharded validation)."""
    from paper_2601_13684_b200._lib import HCError
    from paper_2601_13684_b200.decoder import HeteroCacheDecoder
    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.parallel import assign_units
    from paper_2601_13684_b200.workload import ModelShape, Workload, plan_for

    model = ModelShape("tiny", NL, 32, 8)
    tax, plan = plan_for(Workload("tiny", model, L, B, 0.10, T, 0, layers=NL))
    owned = assign_units(tax, plan, B, 2, T)
    kw = dict(batch=B, group=model.group, max_decode=T, chunk=256)
    with pytest.raises(HCError):
        HeteroCacheDecoder(tax, plan, EngineConfig(), owned=owned[0], recall_topk=64, **kw)
    split = owned[0].copy()
    c = tax.clusters[0]
    split[0, c.satellites[0][0], c.satellites[0][1]] = not split[0, c.pivot[0], c.pivot[1]]
    with pytest.raises(HCError):
        HeteroCacheDecoder(tax, plan, EngineConfig(), owned=split, **kw)
