"""GPU pipeline vs the independent CPU decoder oracle, same inputs end to end.

Both sides generate the workload from the same counter-based generator (the
GPU kernel csrc/synth.cu and its host twin oracle/synth.c, checked bitwise
here), prefill with the observation-window scoring the bench uses, and decode
across planted topic shifts with the bench's own drift / link settings.  The
CPU side (oracle/cpu_decoder.py) computes its own fp32 rows and decisions, so
this checks the whole path at once: K5 prefill rows -> K1 selection, K4
attention, pivot rows, the K1+K2 monitor, fire selection, byte / completion
accounting, landing -- events must be identical and every output within the
stated bf16 tolerance, at every step.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

O_ATOL, O_RTOL = 4e-3, 1e-2


def test_device_generator_matches_host_twin():
    import torch

    from oracle.synth import HostNormal
    from paper_2601_13684_b200.workload import DeviceNormal, stream_key

    for key, off, n in ((stream_key(1, 2, 3), 0, 1 << 20), (stream_key(9), 12345, 777),
                        (2 ** 64 - 5, 2 ** 40, 4096)):
        d = DeviceNormal()((n,), key, off).cpu()
        h = HostNormal()((n,), key, off)
        assert torch.equal(d, h)


def _run_pair(heads, L, NL, B, T, every, obs, bw, c=0.1, chunk=256, seed=20261018,
              delay=1, seqs=None):
    import torch

    from oracle.cpu_decoder import CpuDecoder
    from oracle.synth import HostNormal
    from paper_2601_13684_b200.decoder import HeteroCacheDecoder
    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.workload import (ModelShape, SyntheticKV, Workload, decode_queries,
                                                plan_for, staggered_shifts)

    model = ModelShape("e2e", NL, *heads)
    tax, plan = plan_for(Workload("e2e", model, L, B, c, T, 0, layers=NL))
    cfg = EngineConfig(tau_drift=0.5, window=8, update_delay_steps=delay, transfer_bandwidth=bw)
    shifts = staggered_shifts(B, NL, 2, T, every)
    dec = HeteroCacheDecoder(tax, plan, cfg, batch=B, group=model.group, max_decode=T,
                             chunk=chunk, obs_window=obs, track_sets=True)
    gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=plan.l_base_int,
                      seed=seed)
    for l in range(NL):
        k, v, q = gen.layer_kv(l, obs)
        dec.prefill_layer(l, k, v, q)
        del k, v
    torch.cuda.synchronize()
    dec.finish_prefill()
    qs = decode_queries(gen, T, shifts)
    news = [gen.step_inputs(100 + (t % 4), None)[1:] for t in range(T + 1)]
    outs = {}
    for t in range(1, T + 1):
        o = torch.empty_like(qs[t])
        dec.decode_step(t, qs[t], *news[t], o)
        outs[t] = o.cpu()
    dec.sync()
    seqs = list(range(B)) if seqs is None else seqs
    hgen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=plan.l_base_int,
                       seed=seed, normal=HostNormal(), seqs=seqs)
    hqs = decode_queries(hgen, T, shifts)
    assert torch.equal(hqs.cpu(), qs[:, seqs].cpu())  # same inputs on both sides
    hnews = [hgen.step_inputs(100 + (t % 4), None)[1:] for t in range(T + 1)]
    roles = {hd: p.role for hd, p in tax.heads.items()}
    clusters = [(c_.pivot, tuple(c_.satellites)) for c_ in tax.clusters]
    worst = 0.0
    n_events = 0
    cpu = [CpuDecoder(roles=roles, clusters=clusters, lengths=dict(plan.lengths),
                      l_base_int=plan.l_base_int, prefill_len=L, max_decode=T,
                      group=model.group, transfer_bandwidth=bw, update_delay_steps=delay)
           for _ in seqs]
    for l in range(NL):
        k, v, q = hgen.layer_kv(l, obs)
        for i, cd in enumerate(cpu):
            cd.prefill(l, k[i], v[i], q[i])
    for t in range(1, T + 1):
        for i, (b, cd) in enumerate(zip(seqs, cpu)):
            o_ref, _ = cd.step(t, hqs[t][i], hnews[t][0][i], hnews[t][1][i])
            got = outs[t][b].float()
            err = (got - o_ref).abs()
            assert bool((err <= O_ATOL + O_RTOL * o_ref.abs()).all()), (t, b, float(err.max()))
            worst = max(worst, float(err.max()))
    for i, (b, cd) in enumerate(zip(seqs, cpu)):
        got = [dict(trigger_step=e.trigger_step, pivot=e.pivot, completion_step=e.completion_step,
                    transfer_bytes=e.transfer_bytes, fetches=e.fetches)
               for e in dec.states[b].events]
        assert got == cd.events, f"sequence {b}: GPU events differ from the CPU decoder's"
        n_events += len(got)
        for hd in cd.comp:
            assert np.array_equal(dec.dynamic_set(b, hd), np.sort(cd.dynamic[hd])), (b, hd)
    dec.close()
    return n_events, worst


@pytest.mark.parametrize("kw", [
    dict(heads=(28, 4), L=3000, NL=2, B=2, T=40, every=12, obs=18, bw=1 << 30),
    dict(heads=(32, 8), L=4096, NL=1, B=1, T=40, every=10, obs=32, bw=2 << 20),   # cfg1-like
    dict(heads=(32, 8), L=2500, NL=2, B=2, T=48, every=9, obs=1, bw=150000, delay=2),
])
def test_gpu_pipeline_equals_cpu_decoder(kw):
    n, worst = _run_pair(**kw)
    assert n >= 1, "planted shifts must fire"
    print(f"events {n}, max |O - O_cpu| {worst:.2e}")


def test_gpu_pipeline_equals_cpu_decoder_at_128k():
    """cfg3 shape (Qwen2.5-7B, 5% budget, w = 18 observation window, chunk 1024),
    one of two sequences replayed on the CPU."""
    n, worst = _run_pair(heads=(28, 4), L=131072, NL=2, B=2, T=20, every=9, obs=18,
                         bw=64 << 20, c=0.05, chunk=1024, seqs=[1])
    assert n >= 1
