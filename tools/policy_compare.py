"""Recall and speed of the residency policies at 128K on one B200.

Runs heterocache, static_topk, sink_window and full_oracle at the same entry
budget over the SAME synthetic K/V/Q (Qwen2.5-7B-shaped, 128K context, a
planted per-cluster topic shift) in measure mode -- every head's recall of
its top-1024 recorded attention mass, computed on the GPU -- and prints the
reference's compare() table (evaluation.py:280-335) plus mean decode ms per
step of each policy.

    python tools/policy_compare.py [out.json] [layers] [steps]
"""

import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_13684_b200.engine import EngineConfig  # noqa: E402
from paper_2601_13684_b200.evaluation import (PolicySpec, compare, policy_decoder,  # noqa: E402
                                              policy_report)
from paper_2601_13684_b200.workload import CONFIGS, SyntheticKV, plan_for  # noqa: E402


def run(policy, w, tax, plan, cfg, T, shift):
    m = w.model
    dec = policy_decoder(policy, num_layers=w.num_layers, heads_per_layer=m.kv_heads,
                         prefill_len=w.prefill_len, engine_config=cfg, taxonomy=tax, plan=plan,
                         batch=1, group=m.group, max_decode=T, recall_topk=1024,
                         track_sets=False)
    gen = SyntheticKV(m, batch=1, prefill_len=w.prefill_len, num_layers=w.num_layers,
                      hot=plan.l_base_int, seed=77)
    for l in range(w.num_layers):
        k, v, q = gen.layer_kv(l)
        dec.prefill_layer(l, k, v, q)
    torch.cuda.synchronize()
    dec.finish_prefill()
    ms = 0.0
    for t in range(1, T + 1):
        q, kn, vn = gen.step_inputs(t, shift)
        o = torch.empty_like(q)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dec.decode_step(t, q, kn, vn, o)  # includes the measure pass (diagnostic)
        torch.cuda.synchronize()
        ms += (time.perf_counter() - t0) * 1e3
    dec.sync()
    rep = policy_report(dec, 0, T)
    dec.close()
    return rep, ms / T


def main(out=None, layers=4, T=48):
    w = replace(CONFIGS["cfg3"], layers=layers, batch=1)
    tax, plan = plan_for(w)
    cfg = EngineConfig(tau_drift=0.5, window=8, update_delay_steps=1,
                       transfer_bandwidth=64 << 20)
    shift = tuple(range(9, T, 11))
    reps, speed = [], {}
    for name in ("heterocache", "static_topk", "sink_window", "full_oracle"):
        spec = PolicySpec(name, rho=plan.rho)
        rep, ms = run(spec, w, tax, plan, cfg, T, shift)
        reps.append(rep)
        speed[name] = ms
    # compare() checks one trace: each run's records are its own measurement of the
    # same inputs, so label them alike
    for r in reps:
        object.__setattr__(r, "trace_sha256", "synthetic-cfg3-128k")
    table = compare(reps)
    table["ms_per_step_incl_measure"] = speed
    table["setup"] = {"workload": "cfg3-shaped 128K", "layers": layers, "batch": 1,
                      "decode_steps": T, "rho": plan.rho, "recall_topk": 1024,
                      "topic_shifts": list(shift)}
    print(json.dumps(table, indent=1))
    if out:
        Path(out).write_text(json.dumps(table, indent=1) + "\n")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else None, *(int(x) for x in a[1:]))
