"""Synthetic head profiling for the bench's roles and budgets.

    traces -> run_taxonomy -> plan_budget           (profiling.py:441-454,
                                                      budget.py:211-232)

Calibration traces are decodes of the synthetic model itself (the workload's
shape, a separate seed, shorter prompts) with full caches in measure mode:
every head's dense GQA-mean row per step (K5 on the tensor cores) and its
top-k records, in HCTRACE1 form (tools/export_trace.py), then the taxonomy
(K1 top-k sets, K6 tcgen05 Gram intersection counts) and the stability-
weighted budget at the workload's compression.  The paper profiles on 50
samples of ~10K tokens (tools/calibrate.py runs that scale);
the bench uses a few shorter samples so the profile fits its setup budget.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class CalibSpec:
    samples: int = 4        # calibration prompts
    prefill_len: int = 4096
    steps: int = 16         # decode steps recorded per prompt
    shift_every: int = 6    # planted topic shifts during the calibration decodes
    seed: int = 7000


def profiling_topk(L: int) -> int:
    """metrics.py:109-110 default: min(1000, ceil(L / 10))."""
    return min(1000, -(-L // 10))


def calibration_traces(model, num_layers: int, spec: CalibSpec, batch: int = 4):
    """Measure-mode full-cache decodes -> [(idx, scores, L)] per sample."""
    import torch

    from .engine import EngineConfig
    from .evaluation import PolicySpec, policy_decoder
    from .trace import PAD_INDEX
    from .workload import SyntheticKV, decode_queries, staggered_shifts

    L, T, k = spec.prefill_len, spec.steps, profiling_topk(spec.prefill_len)
    NL, H = num_layers, model.kv_heads
    traces = []
    for first in range(0, spec.samples, batch):
        B = min(batch, spec.samples - first)
        dec = policy_decoder(PolicySpec("full_oracle"), num_layers=NL, heads_per_layer=H,
                             prefill_len=L, engine_config=EngineConfig(), batch=B,
                             group=model.group, max_decode=T, recall_topk=k, track_sets=False)
        gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=k,
                          seed=spec.seed + first)
        for l in range(NL):
            kk, v, q = gen.layer_kv(l)
            dec.prefill_layer(l, kk, v, q)
            del kk, v
        torch.cuda.synchronize()
        dec.finish_prefill()
        qs = decode_queries(gen, T, staggered_shifts(B, NL, 2, T + 1, spec.shift_every))
        idx = np.full((B, T + 1, NL, H, k), PAD_INDEX, dtype=np.uint32)
        sc = np.zeros((B, T + 1, NL, H, k), dtype=np.float32)

        def grab(t):
            for b in range(B):
                for l in range(NL):
                    for h in range(H):
                        idx[b, t, l, h], sc[b, t, l, h] = dec.measure_records(b, (l, h))

        grab(0)
        for t in range(1, T + 1):
            _, kn, vn = gen.step_inputs(t, None)
            o = torch.empty_like(qs[t])
            dec.decode_step(t, qs[t], kn, vn, o, rows=False)
            grab(t)
        dec.close()
        traces += [(idx[b], sc[b], L) for b in range(B)]
    return traces


def calibrate(model, num_layers: int, compression: float, prefill_len: int,
              spec: CalibSpec = CalibSpec()):
    """Profile the synthetic model and plan its budget at compression c
    (L_base = c * L over the profiled compressed heads).  Returns
    (taxonomy, plan, info)."""
    from .budget import BudgetConfig, plan_budget
    from .profiling import ProfileConfig, run_taxonomy
    from .trace import TraceManifest, make_trace

    t0 = time.time()
    raw = calibration_traces(model, num_layers, spec)
    t1 = time.time()
    k = profiling_topk(spec.prefill_len)
    m = TraceManifest(f"calib-{model.name}", num_layers, model.kv_heads, spec.prefill_len,
                      spec.steps, k, 0, 2 * model.head_dim * 2)
    tax = run_taxonomy([make_trace(m, i, s) for i, s, _ in raw], ProfileConfig())
    t2 = time.time()
    n_full = len(tax.full_heads())
    n = len(tax.heads)
    rho = (n_full + compression * (n - n_full)) / n
    plan = plan_budget(tax, BudgetConfig(rho=rho, min_length=16), prefill_len)
    info = summary(tax, plan, spec, t1 - t0, t2 - t1)
    return tax, plan, info


def summary(tax, plan, spec, trace_s, taxonomy_s) -> dict:
    """Role mix and stabilities of a profiled taxonomy (bench config)."""
    roles = sorted(tax.heads.items())
    H = tax.heads_per_layer
    per_layer = [[p.role for (l, h), p in roles if l == ll] for ll in range(tax.num_layers)]
    mixes = {}
    for r in per_layer:
        mixes[",".join(r)] = mixes.get(",".join(r), 0) + 1
    stab = {}
    for (l, h), p in roles:
        stab.setdefault(p.role, []).append(p.s_stable)
    lens = {}
    for hd, n in plan.lengths.items():
        lens.setdefault(tax.heads[hd].role, []).append(n)
    return {
        "source": "profiled: measure-mode decodes of the synthetic model -> run_taxonomy -> "
                  "plan_budget",
        "samples": spec.samples, "prefill_len": spec.prefill_len, "steps": spec.steps,
        "profiling_topk": profiling_topk(spec.prefill_len),
        "role_counts": tax.role_counts(), "clusters": len(tax.clusters),
        "layer_role_mixes": mixes, "heads_per_layer": H,
        "s_stable_by_role": {r: [round(min(v), 4), round(float(np.median(v)), 4),
                                 round(max(v), 4)] for r, v in stab.items()},
        "l_h_by_role": {r: [min(v), int(np.median(v)), max(v)] for r, v in lens.items()},
        "rho": plan.rho, "l_base_int": plan.l_base_int,
        "trace_s": trace_s, "taxonomy_s": taxonomy_s,
    }
