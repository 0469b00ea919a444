"""The CPU decoder oracle (oracle/cpu_decoder.py) against the pinned replay.

CpuDecoder recomputes the rows itself (fp32 attention) and runs the
reference's decision sequence step by step; the bench times it as the CPU
baseline.  Its decisions must equal hc_oracle.replay (pinned to the
reference's own CacheEngine runs, tests/test_oracle.py) over a trace made of
its own rows, and its outputs must be the fp32 attention over exactly the
CacheView resident sets.  Also: the host generator twin reproduces any
sequence subset of the batch.
"""

import numpy as np
import pytest
import torch

from oracle import hc_oracle as O
from oracle.attention_oracle import unit_attention
from oracle.cpu_decoder import CpuDecoder
from oracle.synth import HostNormal
from paper_2601_13684_b200.workload import (ModelShape, SyntheticKV, Workload, decode_queries,
                                            plan_for, staggered_shifts)


def _setup(heads=(16, 4), L=600, NL=2, B=2, T=30, every=10, seed=3, bw=1 << 30, c=0.1):
    model = ModelShape("t", NL, *heads)
    tax, plan = plan_for(Workload("t", model, L, B, c, T, 0, layers=NL))
    gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=plan.l_base_int,
                      seed=seed, normal=HostNormal())
    shifts = staggered_shifts(B, NL, 2, T, every)
    roles = {hd: p.role for hd, p in tax.heads.items()}
    clusters = [(c.pivot, tuple(c.satellites)) for c in tax.clusters]
    return model, tax, plan, gen, shifts, roles, clusters


@pytest.mark.parametrize("kw", [dict(), dict(heads=(32, 8), NL=1, B=1), dict(bw=9000, every=6),
                                dict(heads=(28, 4), L=900, T=24)])
def test_cpu_decoder_decisions_equal_replay_of_its_rows(kw):
    model, tax, plan, gen, shifts, roles, clusters = _setup(**kw)
    T, L, NL, H, B = 30 if "T" not in kw else kw["T"], gen.L, gen.NL, gen.H, gen.B
    bw = kw.get("bw", 1 << 30)
    qs = decode_queries(gen, T, shifts)
    news = [gen.step_inputs(100 + t, None)[1:] for t in range(T + 1)]
    kv = [gen.layer_kv(l, 1) for l in range(NL)]
    fired = 0
    for b in range(B):
        dec = CpuDecoder(roles=roles, clusters=clusters, lengths=dict(plan.lengths),
                         l_base_int=plan.l_base_int, prefill_len=L, max_decode=T,
                         group=model.group, transfer_bandwidth=bw, record_rows=True)
        for l in range(NL):
            k, v, q = kv[l]
            dec.prefill(l, k[b], v[b], q[b])
        outs = {}
        dyn = {}
        for t in range(1, T + 1):
            outs[t], _ = dec.step(t, qs[t][b], news[t][0][b], news[t][1][b])
            dyn[t] = {hd: dec.dynamic[hd] for hd in dec.comp}
        idx = np.full((T + 1, NL, H, L + T), O.PAD_INDEX, dtype=np.uint32)
        sc = np.zeros((T + 1, NL, H, L + T), dtype=np.float32)
        for (l, h), row in dec.rows0.items():
            idx[0, l, h, :L] = np.arange(L)
            sc[0, l, h, :L] = row
        for (t, (l, h)), row in dec.record.items():
            idx[t, l, h, :L + t] = np.arange(L + t)
            sc[t, l, h, :L + t] = row
        ref = O.replay(idx, sc, prefill_len=L, bytes_per_kv_entry=512, roles=roles,
                       clusters=clusters, lengths=dict(plan.lengths), l_base_int=plan.l_base_int,
                       transfer_bandwidth=bw, measure=False, record_dynamic=True)
        assert dec.events == ref["events"]
        fired += len(ref["events"])
        for t in (1, T // 2, T):
            for hd in dec.comp:
                assert set(dyn[t][hd].tolist()) == set(ref["dynamic_trace"][t][hd])
        # outputs: fp32 attention over the CacheView set at step T
        t = T
        G = model.group
        for (l, h) in [(0, 0), (0, 1), (NL - 1, H - 1)]:
            hd = (l, h)
            kk = torch.cat([kv[l][0][b, h]] + [news[s][0][b, l, h][None] for s in range(1, t + 1)])
            vv = torch.cat([kv[l][1][b, h]] + [news[s][1][b, l, h][None] for s in range(1, t + 1)])
            base = None if hd in dec.full else ref["dynamic_trace"][t][hd]
            res = sorted(O.resident_positions(L, t, base, 4, 8))
            o_ref, _ = unit_attention(qs[t][b, l, h * G:(h + 1) * G], kk, vv,
                                      None if base is None else res)
            assert torch.allclose(outs[t][l, h * G:(h + 1) * G], o_ref, atol=1e-6, rtol=1e-5)
    assert fired >= 1


def test_host_generator_sequence_subsets_match_full_batch():
    model = ModelShape("t", 2, 32, 8)
    full = SyntheticKV(model, batch=3, prefill_len=700, num_layers=2, hot=40, seed=11,
                       normal=HostNormal())
    part = SyntheticKV(model, batch=3, prefill_len=700, num_layers=2, hot=40, seed=11,
                       normal=HostNormal(), seqs=[2, 0])
    for a, b in zip(full.layer_kv(1, 8), part.layer_kv(1, 8)):
        assert torch.equal(a[[2, 0]], b)
    for a, b in zip(full.step_inputs(4, 2), part.step_inputs(4, 2)):
        assert torch.equal(a[[2, 0]], b)
    sh = staggered_shifts(3, 2, 1, 12, 5)
    assert torch.equal(decode_queries(full, 6, sh)[:, [2, 0]], decode_queries(part, 6, sh))
