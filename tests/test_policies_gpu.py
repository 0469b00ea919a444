"""Baseline residency policies on the GPU.

* Trace mode: ``evaluation.run_policy`` serves full_oracle / static_topk /
  sink_window through the GPU trace engine; every report must equal the
  reference's own ``heterocache.evaluation.run_policy`` report
  (tests/golden/policy_cases.json, made by tests/golden/make_golden.py),
  recall included, refusals included.
* Tensor mode: the same policies served over real K/V by the decoder in
  measure mode; replaying its records through the oracle's run_policy
  restatement (pinned to the reference in test_oracle.py) gives the same
  StepRows.
"""

import numpy as np
import pytest

from golden_io import case_arrays, engine_cases, policy_cases, policy_kwargs
from oracle import hc_oracle as O

pytestmark = pytest.mark.gpu


def _trace(name):
    from paper_2601_13684_b200.trace import TraceManifest, make_trace

    case = next(c for c in engine_cases() if c["name"] == name)
    idx, sc = case_arrays(name)
    return make_trace(TraceManifest(**case["manifest"]), idx, sc)


def test_run_policy_matches_reference_reports():
    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.evaluation import EvaluationError, PolicySpec, run_policy

    n = 0
    for pc in policy_cases():
        tr = _trace(pc["trace"])
        spec = PolicySpec(pc["policy"], rho=pc["rho"], sink_count=pc["sink_count"],
                          window=pc["window"])
        ecfg = None if pc["engine"] is None else EngineConfig(**pc["engine"])
        exp = pc["expected"]
        if "error" in exp:
            with pytest.raises(EvaluationError):
                run_policy(tr, spec, engine_config=ecfg)
            continue
        got = run_policy(tr, spec, engine_config=ecfg).to_json_dict()
        assert got == exp, (pc["trace"], pc["policy"], pc["rho"])
        n += 1
    assert n >= 60


def test_compare_orders_policies_and_checks_budgets():
    from paper_2601_13684_b200.evaluation import (BudgetMismatchError, PolicySpec, compare,
                                                  run_policies)

    tr = _trace("drift_seed5")
    reps = run_policies(tr, [PolicySpec("static_topk", rho=0.3),
                             PolicySpec("sink_window", rho=0.3), PolicySpec("full_oracle")])
    table = compare(reps)
    assert [r["policy"] for r in table["policies"]] == ["full_oracle", "sink_window",
                                                        "static_topk"]
    assert table["policies"][0]["mean_recall"] == 1.0
    with pytest.raises(BudgetMismatchError):
        run_policies(tr, [PolicySpec("static_topk", rho=0.3), PolicySpec("sink_window", rho=0.6)])


@pytest.mark.parametrize("name,kw", [
    ("static_topk", dict(rho=0.2)),
    ("sink_window", dict(rho=0.15)),          # recency window 101 > 32: contiguous tail block
    ("sink_window", dict(rho=0.3, sink_count=0)),
    ("full_oracle", dict()),
])
def test_tensor_mode_policies_match_oracle(name, kw):
    import torch

    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.evaluation import PolicySpec, policy_decoder, policy_report
    from paper_2601_13684_b200.workload import ModelShape, SyntheticKV

    B, NL, L, T = 2, 2, 700, 20
    model = ModelShape("tiny-qwen", NL, 16, 4)
    spec = PolicySpec(name, **kw)
    ecfg = EngineConfig(sink_count=4, recency_window=8)
    dec = policy_decoder(spec, num_layers=NL, heads_per_layer=model.kv_heads, prefill_len=L,
                         engine_config=ecfg, batch=B, group=model.group, max_decode=T,
                         chunk=256, recall_topk=64)
    gen = SyntheticKV(model, batch=B, prefill_len=L, num_layers=NL, hot=64, seed=5)
    for l in range(NL):
        k, v, q = gen.layer_kv(l)
        dec.prefill_layer(l, k, v, q)
    torch.cuda.synchronize()
    dec.finish_prefill()
    H = model.kv_heads
    K = dec.record_k
    idx = np.full((B, T + 1, NL, H, K), O.PAD_INDEX, dtype=np.uint32)
    sc = np.zeros((B, T + 1, NL, H, K), dtype=np.float32)

    def grab(t):
        for b in range(B):
            for l in range(NL):
                for h in range(H):
                    idx[b, t, l, h], sc[b, t, l, h] = dec.measure_records(b, (l, h))

    grab(0)
    for t in range(1, T + 1):
        q, kn, vn = gen.step_inputs(t, 9)
        o = torch.empty_like(q)
        dec.decode_step(t, q, kn, vn, o)
        grab(t)
    dec.sync()
    pc = {"policy": name, "rho": spec.rho, "sink_count": spec.sink_count, "window": spec.window,
          "engine": {"sink_count": 4, "recency_window": 8}}
    for b in range(B):
        ref = O.static_policy_report(idx[b], sc[b], **policy_kwargs(pc, L))
        rep = policy_report(dec, b, T)
        assert rep.policy == name and rep.update_delay_steps == 0 and rep.events == ()
        assert rep.budget_ceiling == ref["budget_ceiling"]
        got = [r.to_json_dict() for r in rep.rows]
        assert got == ref["rows"], (b, name)
    if name == "sink_window":  # only sinks + window + appends are resident
        want = B * NL * H * (spec.sink_count + spec.effective_window(L))
        assert dec.resident_rows(T) == want
