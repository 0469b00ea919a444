"""CPU restatement of the bench's synthetic profiling -- TEST / BASELINE INFRASTRUCTURE.

Same calibration workload as paper_2601_13684_b200/calibration.py (same
counter-based inputs through oracle/synth.py), with every head's full-cache
GQA-mean rows in fp32 on the host cores (model.ts:274-291; step 0 the last
prompt token, export.ts:125-127), top-k records (metrics.py:42-45 order),
then the pinned restatements hc_oracle.run_taxonomy (profiling.py:253-454) and
hc_oracle.plan_budget (budget.py:211-232).  Used by bench.py's reference arm.
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch

from . import hc_oracle as O
from .synth import HostNormal


def _row(q, k, G):
    s = (q.float() @ k.float().T) * (1.0 / math.sqrt(k.shape[-1]))
    p = torch.softmax(s, dim=-1)
    acc = p[0].clone()
    for j in range(1, G):
        acc = acc + p[j]
    return (acc / G).numpy()


def calibration_traces(model, num_layers, spec):
    from paper_2601_13684_b200.calibration import profiling_topk
    from paper_2601_13684_b200.workload import SyntheticKV, decode_queries, staggered_shifts

    L, T, k = spec.prefill_len, spec.steps, profiling_topk(spec.prefill_len)
    NL, H, G = num_layers, model.kv_heads, model.group
    traces = []
    batch = 4
    for first in range(0, spec.samples, batch):
        B = min(batch, spec.samples - first)
        gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=k,
                          seed=spec.seed + first, normal=HostNormal())
        qs = decode_queries(gen, T, staggered_shifts(B, NL, 2, T + 1, spec.shift_every))
        news = [gen.step_inputs(t, None) for t in range(1, T + 1)]
        idx = np.full((B, T + 1, NL, H, k), O.PAD_INDEX, dtype=np.uint32)
        sc = np.zeros((B, T + 1, NL, H, k), dtype=np.float32)
        for l in range(NL):
            kk, vv, q0 = gen.layer_kv(l)
            for b in range(B):
                for h in range(H):
                    keys = torch.cat([kk[b, h]] + [news[t][1][b, l, h][None] for t in range(T)])
                    rows = [_row(q0[b, h * G:(h + 1) * G], keys[:L], G)]
                    for t in range(1, T + 1):
                        rows.append(_row(qs[t][b, l, h * G:(h + 1) * G], keys[:L + t], G))
                    for t, r in enumerate(rows):
                        sel = O.top_k_dense(r, k)
                        idx[b, t, l, h, :len(sel)] = sel
                        sc[b, t, l, h, :len(sel)] = r[sel]
        traces += [(idx[b], sc[b], L) for b in range(B)]
    return traces


def calibrate(model, num_layers, compression, prefill_len, spec):
    """(roles, clusters, lengths, l_base_int, s_stable, seconds)."""
    t0 = time.time()
    traces = calibration_traces(model, num_layers, spec)
    roles, _, clusters, s_stable, _ = O.run_taxonomy(traces)
    n_full = sum(r in ("pivot", "volatile") for r in roles.values())
    n = len(roles)
    rho = (n_full + compression * (n - n_full)) / n
    plan = O.plan_budget(roles, s_stable, rho=rho, prefill_len=prefill_len)
    return roles, clusters, plan["lengths"], plan["l_base_int"], rho, s_stable, time.time() - t0
