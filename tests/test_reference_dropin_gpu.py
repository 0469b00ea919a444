"""The reference package itself, with the B200 engine dropped in.

The unmodified reference (`heterocache`, installed offline into baseline/_ref
with `pip install --no-index --no-deps --target baseline/_ref`, git-ignored,
shipped with the gpurun snapshot) generates its own synthetic traces
(synthetic.generate_synthetic), profiles them (profiling.run_taxonomy) and
plans budgets (budget.plan_budget).  `heterocache.evaluation.run_policy` is then
run twice on the reference's own objects: stock, and with
`heterocache.engine.run_simulation` patched to construct
`paper_2601_13684_b200.engine.CacheEngine` exactly as INTEGRATION.md shows.
The reports must be identical (JSON dicts: every StepRow incl. recall, every
RetrievalRecord, aggregates).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "heterocache").exists(),
                                 reason="reference not installed into baseline/_ref")]


@pytest.fixture(scope="module")
def hc():
    sys.path.insert(0, str(REF))
    import heterocache.budget as budget
    import heterocache.engine as engine
    import heterocache.evaluation as evaluation
    import heterocache.profiling as profiling
    import heterocache.synthetic as synthetic

    assert str(REF) in engine.__file__  # the installed reference, not this repo
    return dict(budget=budget, engine=engine, evaluation=evaluation, profiling=profiling,
                synthetic=synthetic)


def _spec(hc, seed, *, layers=2, heads=6, prefill_len=120, decode_steps=40, shift=True):
    S = hc["synthetic"]
    arch, clusters = {}, {}
    for layer in range(layers):
        arch[(layer, 0)] = S.StableHead(hot_size=12, noise_rate=0.05)
        arch[(layer, 1)] = S.DecayingHead(hot_size=12, drift_rate=0.35)
        for head in range(2, heads):
            arch[(layer, head)] = S.ClusterMember(layer, 0.9)
        clusters[layer] = S.ClusterSpec(hot_size=24)
    events = tuple(S.DriftEvent(step=decode_steps // 2, heads=((l, 2),), replace_fraction=0.8)
                   for l in range(layers)) if shift else ()
    return S.SynthSpec(num_layers=layers, heads_per_layer=heads, prefill_len=prefill_len,
                       decode_steps=decode_steps, trace_topk=40, archetypes=arch,
                       clusters=clusters, drift_events=events, seed=seed)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("policy", ["heterocache", "no_allocation", "no_retrieval"])
def test_run_policy_with_b200_engine_patched_in(hc, seed, policy, monkeypatch):
    from paper_2601_13684_b200.engine import CacheEngine as B200Engine

    ev, eng = hc["evaluation"], hc["engine"]
    trace, _ = hc["synthetic"].generate_synthetic(_spec(hc, 100 + seed))
    taxonomy = hc["profiling"].run_taxonomy([trace], hc["profiling"].ProfileConfig())
    rho = 0.4
    plan = hc["budget"].plan_budget(taxonomy, hc["budget"].BudgetConfig(rho=rho, min_length=4),
                                    trace.manifest.prefill_len)
    rng = np.random.default_rng(seed)
    cfg = eng.EngineConfig(window=int(rng.choice([4, 8])),
                           update_delay_steps=int(rng.integers(1, 4)),
                           transfer_bandwidth=int(rng.choice([3000, 1 << 30])),
                           eval_every_step=bool(seed % 2))
    spec = ev.PolicySpec(policy, rho=rho)
    stock = ev.run_policy(trace, spec, taxonomy=taxonomy, plan=plan, engine_config=cfg)

    calls = []

    def run_simulation(trace, taxonomy, plan, config=eng.EngineConfig()):
        calls.append(1)
        return B200Engine(trace, taxonomy, plan, config).run()

    monkeypatch.setattr(eng, "run_simulation", run_simulation)
    b200 = ev.run_policy(trace, spec, taxonomy=taxonomy, plan=plan, engine_config=cfg)
    assert calls, "run_policy must go through the patched engine"
    assert b200.to_json_dict() == stock.to_json_dict()
    if policy == "heterocache" and seed == 0:
        assert stock.events, "the planted drift must fire at least once"
