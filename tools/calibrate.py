"""Offline calibration at the paper's scale on one B200.

The paper profiles heads on 50 calibration samples of ~10K tokens
(PAPER.md:497).  This tool runs that flow end to end on the GPU:

  1. every sample is decoded with full caches (full_oracle policy) in measure
     mode, so each head's dense attention row per step becomes top-k trace
     records (K5 rows, K1 selection, records in HCTRACE1 order);
  2. profiling.run_taxonomy over all samples' traces: K1 top-k sets and K6
     tcgen05 Gram matrices per (trace, layer), vectorised medians;
  3. plan_budget on the resulting taxonomy.

On the synthetic workload (planted cluster per layer: pivot + satellites
sharing hot sets, anchors with their own steady topic, volatile heads
diffuse) the recovered roles are compared with the planted ones.

    python tools/calibrate.py [out.json] [samples] [prefill] [steps]
"""

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_13684_b200.budget import BudgetConfig, plan_budget  # noqa: E402
from paper_2601_13684_b200.engine import EngineConfig  # noqa: E402
from paper_2601_13684_b200.evaluation import PolicySpec, policy_decoder  # noqa: E402
from paper_2601_13684_b200.profiling import ProfileConfig, run_taxonomy  # noqa: E402
from paper_2601_13684_b200.trace import PAD_INDEX, TraceManifest, make_trace  # noqa: E402
from paper_2601_13684_b200.workload import LLAMA3_8B, SyntheticKV  # noqa: E402


def sample_traces(model, n, L, T, batch, k, seed0):
    """n traces [T+1, NL, H, k] of full-cache decodes, `batch` samples per decoder."""
    import numpy as np

    NL, H = model.num_layers, model.kv_heads
    traces = []
    for first in range(0, n, batch):
        B = min(batch, n - first)
        dec = policy_decoder(PolicySpec("full_oracle"), num_layers=NL, heads_per_layer=H,
                             prefill_len=L, engine_config=EngineConfig(), batch=B,
                             group=model.group, max_decode=T, recall_topk=k, track_sets=False)
        gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=k,
                          seed=seed0 + first)
        for l in range(NL):
            kk, v, q = gen.layer_kv(l)
            dec.prefill_layer(l, kk, v, q)
        torch.cuda.synchronize()
        dec.finish_prefill()
        idx = np.full((B, T + 1, NL, H, k), PAD_INDEX, dtype=np.uint32)
        sc = np.zeros((B, T + 1, NL, H, k), dtype=np.float32)

        def grab(t):
            for b in range(B):
                for l in range(NL):
                    for h in range(H):
                        idx[b, t, l, h], sc[b, t, l, h] = dec.measure_records(b, (l, h))

        grab(0)
        for t in range(1, T + 1):
            q, kn, vn = gen.step_inputs(t, None)
            o = torch.empty_like(q)
            dec.decode_step(t, q, kn, vn, o, rows=False)
            grab(t)
        dec.close()
        m = TraceManifest(f"calib-{model.name}", NL, H, L, T, k, 0, 2 * model.head_dim * 2)
        traces += [make_trace(m, idx[b], sc[b]) for b in range(B)]
    return traces


def main(out=None, n=50, L=10240, T=32, batch=10):
    model = LLAMA3_8B
    k = min(1000, -(-L // 10))  # metrics.py default_profiling_topk
    t0 = time.time()
    traces = sample_traces(model, n, L, T, batch, k, seed0=1000)
    t1 = time.time()
    tax = run_taxonomy(traces, ProfileConfig())
    t2 = time.time()
    # the budget at c = 10% of the compressed heads' prefill
    n_full = len(tax.full_heads())
    rho = (n_full + 0.10 * (len(tax.heads) - n_full)) / len(tax.heads)
    plan = plan_budget(tax, BudgetConfig(rho=rho, min_length=16), L)
    planted = model.layer_roles()
    got = {(l, h): p.role for (l, h), p in tax.heads.items()}
    match = sum(got[(l, h)] == planted[h] for (l, h) in got)
    res = {"samples": n, "prefill_len": L, "decode_steps": T, "profiling_topk": k,
           "model": model.name, "trace_seconds": t1 - t0, "taxonomy_seconds": t2 - t1,
           "role_counts": tax.role_counts(), "clusters": len(tax.clusters),
           "planted_roles_per_layer": list(planted),
           "roles_matching_planted": f"{match}/{len(got)}",
           "rho": rho, "l_base_int": plan.l_base_int,
           "role_confusion": {f"{a}->{b}": sum(1 for (l, h), r in got.items()
                                               if planted[h] == a and r == b)
                              for a in sorted(set(planted)) for b in sorted(set(got.values()))
                              if any(planted[h] == a and r == b for (l, h), r in got.items())}}
    print(json.dumps(res, indent=1))
    if out:
        Path(out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else None, *(int(x) for x in a[1:]))
