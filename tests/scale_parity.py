"""Output and selection parity at the benchmarked context lengths (helper).

Runs the tensor-mode decoder on a cfg3-shaped (Qwen2.5-7B, 128K, chunk 1024)
or cfg5-shaped (Llama-3.1-8B, 224K) slice across a planted topic shift, so the
run holds a fire and a landing, and checks against the fp32 CPU oracle over
the same bf16 inputs:

  * attention outputs O of every unit of every role (pivot, satellite,
    anchor, volatile) at sampled steps -- always including each landing step,
    where a satellite first serves its fetched set -- over exactly the
    CacheView resident set (engine.py:98-115) the GPU holds at that step;
  * pivot probability rows against the GQA-mean row (model.ts:274-291);
  * the event log against the oracle replay of the GPU's own rows (decisions
    bit-exact given the rows, SURVEY.md section 8c protocol 2);
  * selection precision: at every step, for every pivot and every k the
    engine selects with (l_base for K_base / the overlap, l_s of each
    satellite for fetches; engine.py:232-240, 326-329), the symmetric
    difference between the top-k set of the GPU row and of the oracle's fp32
    and fp64 rows over the same K/V/Q (metrics.py:42-45 order).

Used by tests/test_scale_parity_gpu.py and tools/selection_precision.py.
Test infrastructure: imports the oracle.
"""

from __future__ import annotations

import math

import numpy as np

from oracle import hc_oracle as O
from oracle.attention_oracle import gqa_mean_row, unit_attention

# Stated output tolerance (bf16 K/V/Q in, fp32 accumulation, bf16 P in the PV
# product, bf16 O out): |O - O_ref| <= O_ATOL + O_RTOL * |O_ref| elementwise.
O_ATOL = 4e-3
O_RTOL = 1e-2
# pivot rows (fp32 material): fp32 exp2 / sum rounding vs the oracle's exp
ROW_ATOL = 1e-9
ROW_RTOL = 2e-5

SHAPES = {
    # cfg3: Qwen2.5-7B-shaped, 128K context, 5% budget, split-K chunk 1024
    "cfg3": dict(heads=(28, 4), L=131072, compression=0.05),
    # cfg5: Llama-3.1-8B-shaped, 224K context, 10% budget
    "cfg5": dict(heads=(32, 8), L=229376, compression=0.10),
    # cfg4: R1-Distill-Llama-8B-shaped, 64K prompt, 10% budget (frequent drift)
    "cfg4": dict(heads=(32, 8), L=65536, compression=0.10),
}


def build(shape: str, *, B: int, NL: int, T: int = 24, shift=9, window: int = 8,
          chunk: int = 1024, seed: int = 5, score_material: str = "fp32",
          bandwidth: int = 1 << 30, delay: int = 1, eval_every_step: bool = False):
    import torch

    from paper_2601_13684_b200.decoder import HeteroCacheDecoder
    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.workload import ModelShape, SyntheticKV, Workload, plan_for

    sp = SHAPES[shape]
    model = ModelShape(shape, NL, *sp["heads"])
    L = sp["L"]
    w = Workload(shape, model, L, B, sp["compression"], T, 0, layers=NL)
    tax, plan = plan_for(w)
    cfg = EngineConfig(tau_drift=0.5, window=window, update_delay_steps=delay,
                       transfer_bandwidth=bandwidth, eval_every_step=eval_every_step)
    dec = HeteroCacheDecoder(tax, plan, cfg, batch=B, group=model.group, max_decode=T,
                             chunk=chunk, host_pool=True, obs_window=1,
                             score_material=score_material)
    gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=plan.l_base_int,
                      seed=seed)
    dump = torch.zeros(NL, B * model.kv_heads, L, device="cuda")
    dec.lib.hc_engine_set_prefill_dump(dec.handle, dump.data_ptr())
    kv = []
    for l in range(NL):
        k, v, q = gen.layer_kv(l, 1)
        dec.prefill_layer(l, k, v, q)
        kv.append((k.cpu(), v.cpu(), q.cpu()))  # bf16 host copies for the oracle
        del k, v
    torch.cuda.synchronize()
    dec.finish_prefill()
    return dict(dec=dec, gen=gen, kv=kv, dump=dump.cpu().numpy(), tax=tax, plan=plan, cfg=cfg,
                model=model, B=B, NL=NL, L=L, T=T, shift=shift, shape=shape)


def run(ctx):
    """Decode T steps; keep every step's O, pivot rows, appends and dynamic sets."""
    import torch

    dec, gen = ctx["dec"], ctx["gen"]
    B, L, T = ctx["B"], ctx["L"], ctx["T"]
    rows, outs, news, dyn = {}, {}, [], {}
    for t in range(1, T + 1):
        q, kn, vn = gen.step_inputs(t, ctx["shift"])
        o = torch.empty_like(q)
        dec.decode_step(t, q, kn, vn, o)
        news.append((q.cpu(), kn.cpu(), vn.cpu()))
        outs[t] = o.cpu()
        for b in range(B):
            for p in dec.pivots:
                buf = torch.empty(L + t, device="cuda")
                dec.pivot_row(b, p, t, buf)
                rows[(b, p, t)] = buf.cpu().numpy()
        # the sets in force at t (this step's landings applied; a boundary
        # decision stays open until step t+1, as in the bench)
        dyn[t] = {(b, hd): dec.dynamic_set(b, hd) for b in range(B) for hd in dec.comp}
    dec.finish()
    dec.sync()
    ctx.update(rows=rows, outs=outs, news=news, dyn=dyn)
    return ctx


def oracle_replay(ctx, b):
    dec, L, T, NL = ctx["dec"], ctx["L"], ctx["T"], ctx["NL"]
    H = ctx["model"].kv_heads
    K = L + T
    idx = np.full((T + 1, NL, H, K), O.PAD_INDEX, dtype=np.uint32)
    sc = np.zeros((T + 1, NL, H, K), dtype=np.float32)
    for l in range(NL):
        for h in range(H):
            idx[0, l, h, :L] = np.arange(L)
            sc[0, l, h, :L] = ctx["dump"][l, b * H + h]
    for t in range(1, T + 1):
        for p in dec.pivots:
            idx[t, p[0], p[1], :L + t] = np.arange(L + t)
            sc[t, p[0], p[1], :L + t] = ctx["rows"][(b, p, t)]
    roles = {hd: pr.role for hd, pr in ctx["tax"].heads.items()}
    clusters = [(c.pivot, tuple(c.satellites)) for c in ctx["tax"].clusters]
    cfg = ctx["cfg"]
    return O.replay(idx, sc, prefill_len=L, bytes_per_kv_entry=512, roles=roles,
                    clusters=clusters, lengths=dict(ctx["plan"].lengths),
                    l_base_int=ctx["plan"].l_base_int, tau_drift=cfg.tau_drift,
                    window=cfg.window, transfer_bandwidth=cfg.transfer_bandwidth,
                    update_delay_steps=cfg.update_delay_steps, sink_count=cfg.sink_count,
                    recency_window=cfg.recency_window, variant=cfg.variant,
                    eval_every_step=cfg.eval_every_step, measure=False, record_dynamic=True)


def check_events(ctx):
    """GPU events / dynamic sets == oracle replay of the GPU rows, per sequence."""
    dec = ctx["dec"]
    events = []
    for b in range(ctx["B"]):
        ref = oracle_replay(ctx, b)
        got = [dict(trigger_step=e.trigger_step, pivot=e.pivot, completion_step=e.completion_step,
                    transfer_bytes=e.transfer_bytes, fetches=e.fetches)
               for e in dec.states[b].events]
        assert got == ref["events"], f"sequence {b}: event log differs from the oracle replay"
        for t in range(1, ctx["T"] + 1):
            for hd in dec.comp:
                assert set(ctx["dyn"][t][(b, hd)].tolist()) == set(ref["dynamic_trace"][t][hd]), \
                    (b, t, hd)
        events += [(b, e) for e in got]
    return events


def _unit_kv(ctx, b, l, h, t):
    """Position-indexed bf16 K/V [L+t, d] of one unit (prefill + appends)."""
    import torch

    k, v, _ = ctx["kv"][l]
    news = ctx["news"]
    ks = [k[b, h]] + [news[s][1][b, l, h][None] for s in range(t)]
    vs = [v[b, h]] + [news[s][2][b, l, h][None] for s in range(t)]
    return torch.cat(ks), torch.cat(vs)


def _attn64(q, k, v, positions=None):
    import torch

    q, k, v = q.double(), k.double(), v.double()
    if positions is not None:
        pos = torch.as_tensor(positions, dtype=torch.long)
        k, v = k.index_select(0, pos), v.index_select(0, pos)
    s = (q @ k.T) / math.sqrt(q.shape[-1])
    p = torch.softmax(s, dim=-1)
    return p @ v, p


def check_outputs(ctx, steps):
    """O of every unit at `steps` vs the fp32 oracle over the GPU's resident set;
    pivot rows vs the GQA-mean oracle row.  Returns error statistics."""
    dec, cfg = ctx["dec"], ctx["cfg"]
    L, H, G = ctx["L"], ctx["model"].kv_heads, ctx["model"].group
    roles = {hd: pr.role for hd, pr in ctx["tax"].heads.items()}
    st = dict(max_abs=0.0, max_rel=0.0, units=0, row_max_abs=0.0, row_max_rel=0.0, rows=0,
              by_role={}, violations=[])
    for t in steps:
        o = ctx["outs"][t]
        q_t = ctx["news"][t - 1][0]
        for b in range(ctx["B"]):
            for l in range(ctx["NL"]):
                for h in range(H):
                    hd = (l, h)
                    base = None if hd in dec.full else ctx["dyn"][t][(b, hd)].tolist()
                    res = sorted(O.resident_positions(L, t, base, cfg.sink_count,
                                                      cfg.recency_window))
                    kk, vv = _unit_kv(ctx, b, l, h, t)
                    q = q_t[b, l, h * G:(h + 1) * G]
                    o_ref, p = unit_attention(q, kk, vv, None if base is None else res)
                    got = o[b, l, h * G:(h + 1) * G].float()
                    err = (got - o_ref).abs()
                    bound = O_ATOL + O_RTOL * o_ref.abs()
                    ea, er = float(err.max()), float((err / o_ref.abs().clamp_min(1e-3)).max())
                    st["max_abs"] = max(st["max_abs"], ea)
                    st["max_rel"] = max(st["max_rel"], er)
                    st["units"] += 1
                    r = st["by_role"].setdefault(roles[hd], dict(units=0, max_abs=0.0))
                    r["units"] += 1
                    r["max_abs"] = max(r["max_abs"], ea)
                    if not bool((err <= bound).all()):
                        st["violations"].append((t, b, hd, ea))
                    if hd in dec.pivots:
                        row_ref = gqa_mean_row(p).numpy()
                        row = ctx["rows"][(b, hd, t)]
                        d = np.abs(row.astype(np.float64) - row_ref)
                        st["row_max_abs"] = max(st["row_max_abs"], float(d.max()))
                        st["row_max_rel"] = max(st["row_max_rel"], float(
                            (d / np.maximum(np.abs(row_ref), 1e-30)).max()))
                        st["rows"] += 1
                        if not np.allclose(row, row_ref, atol=ROW_ATOL, rtol=ROW_RTOL):
                            st["violations"].append((t, b, hd, "row", float(d.max())))
    return st


def _sym(a, b) -> int:
    return int(np.setxor1d(a, b, assume_unique=True).size // 2)


def selection_precision(ctx, steps=None):
    """Per (step, sequence, pivot, k): |top_k(GPU row) ^ top_k(oracle row)| / 2 for
    the fp32 and fp64 oracle rows, and fp32 vs fp64 (the oracle's own floor)."""
    dec = ctx["dec"]
    G = ctx["model"].group
    plan = ctx["plan"]
    steps = steps or range(1, ctx["T"] + 1)
    out = []
    for t in steps:
        q_t = ctx["news"][t - 1][0]
        for b in range(ctx["B"]):
            for p in dec.pivots:
                l, h = p
                kk, vv = _unit_kv(ctx, b, l, h, t)
                q = q_t[b, l, h * G:(h + 1) * G]
                _, p32 = unit_attention(q, kk, vv)
                _, p64 = _attn64(q, kk, vv)
                r32 = gqa_mean_row(p32).numpy()
                r64 = (p64.sum(0) / G).numpy()
                gpu = ctx["rows"][(b, p, t)]
                ks = [("l_base", plan.l_base_int)] + [
                    (f"sat{s}", dec.effective_length(s)) for s in dec.satellites_of[p]]
                for name, k in ks:
                    k = min(k, ctx["L"] + t)
                    sg = O.top_k_dense(gpu, k)
                    s32 = O.top_k_dense(r32, k)
                    s64 = O.top_k_dense(r64, k)
                    out.append(dict(step=t, seq=b, pivot=list(p), sel=name, k=int(k),
                                    gpu_vs_fp32=_sym(sg, s32), gpu_vs_fp64=_sym(sg, s64),
                                    fp32_vs_fp64=_sym(s32, s64)))
    return out


def summarise(sel):
    keys = ("gpu_vs_fp32", "gpu_vs_fp64", "fp32_vs_fp64")
    res = {"selections": len(sel)}
    for k in keys:
        v = [x[k] for x in sel]
        res[k] = dict(max=max(v) if v else 0, total=int(sum(v)),
                      nonzero=int(sum(1 for x in v if x)))
    return res
