"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference is mounted read-only at
/root/reference and does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Everything written here is produced by the reference's own code
(heterocache.synthetic / profiling / budget / engine / metrics) so the oracle
(oracle/hc_oracle.py) and the CUDA path are pinned to the reference's
outputs, not to our reading of it.  Outputs:

  engine_cases.json / engine_traces.npz   reference CacheEngine runs
  topk_cases.json                          reference top_k_indices answers
  budget_cases.json                        reference plan_budget / allocate
  taxonomy_cases.json                      reference run_taxonomy results
  policy_cases.json                        reference run_policy reports of the
                                           baseline policies (evaluation.py)
  golden_replay.json                       the reference's own golden file
"""

from __future__ import annotations

import json
import os
import shutil
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
sys.dont_write_bytecode = True

from heterocache.budget import BudgetConfig, allocate, plan_budget  # noqa: E402
from heterocache.engine import CacheEngine, EngineConfig  # noqa: E402
from heterocache.evaluation import PolicySpec, run_policy  # noqa: E402
from heterocache.metrics import top_k_indices  # noqa: E402
from heterocache.profiling import (  # noqa: E402
    Cluster, HeadProfile, ProfileConfig, TaxonomyResult, run_taxonomy,
)
from heterocache.synthetic import (  # noqa: E402
    ClusterMember, ClusterSpec, DecayingHead, DriftEvent, StableHead, SynthSpec,
    generate_synthetic, synth_spec_from_json,
)
from heterocache.trace import PAD_INDEX, TraceManifest, make_trace  # noqa: E402

OUT = Path(__file__).resolve().parent


def hid(h):
    return f"{h[0]},{h[1]}"


def drift_spec(seed=5, drift_step=17, replace=0.9, decode_steps=40, topk=96, hot=96):
    # mirrors pkg/tests/test_engine.py:28-52
    return SynthSpec(
        num_layers=1, heads_per_layer=4, prefill_len=400, decode_steps=decode_steps,
        trace_topk=topk,
        archetypes={
            (0, 0): StableHead(hot_size=24, noise_rate=0.05),
            (0, 1): ClusterMember(cluster_id=0, agreement_rate=0.95),
            (0, 2): ClusterMember(cluster_id=0, agreement_rate=0.95),
            (0, 3): DecayingHead(hot_size=24, drift_rate=0.3),
        },
        clusters={0: ClusterSpec(hot_size=hot, drift_rate=0.0)},
        drift_events=(DriftEvent(step=drift_step, heads=((0, 1),), replace_fraction=replace),)
        if drift_step else (),
        seed=seed,
    )


CLUSTER_HOT = {40: 18, 60: 28, 80: 38}


def mixed_spec(seed, *, prefill_len=60, decode_steps=48, shift_step=12, replace=0.9,
               agreement=0.9):
    # mirrors pkg/tests/test_acceptance.py:58-81
    hot = CLUSTER_HOT[prefill_len]
    vh = min(24, hot)
    arch = {
        (0, 0): StableHead(hot_size=6), (0, 1): StableHead(hot_size=6),
        (0, 2): ClusterMember(0, agreement), (0, 3): ClusterMember(0, agreement),
        (0, 4): ClusterMember(0, agreement), (0, 5): ClusterMember(0, agreement),
        (0, 6): DecayingHead(vh, 0.3), (0, 7): DecayingHead(vh, 0.3),
    }
    events = ()
    if shift_step is not None:
        events = (DriftEvent(step=shift_step, heads=((0, 2),), replace_fraction=replace),)
    return SynthSpec(num_layers=1, heads_per_layer=8, prefill_len=prefill_len,
                     decode_steps=decode_steps, trace_topk=hot + 4, archetypes=arch,
                     clusters={0: ClusterSpec(hot_size=hot)}, drift_events=events, seed=seed)


def multi_layer_spec(seed):
    """Two layers x 8 heads, two clusters per layer, drifts in both layers."""
    arch, clusters = {}, {}
    cid = 0
    for layer in range(2):
        arch[(layer, 0)] = StableHead(hot_size=10, noise_rate=0.05)
        arch[(layer, 1)] = DecayingHead(hot_size=20, drift_rate=0.3)
        for head in (2, 3, 4):
            arch[(layer, head)] = ClusterMember(cid, 0.95)
        clusters[cid] = ClusterSpec(hot_size=40)
        for head in (5, 6, 7):
            arch[(layer, head)] = ClusterMember(cid + 1, 0.95)
        clusters[cid + 1] = ClusterSpec(hot_size=40, drift_rate=0.02)
        cid += 2
    events = (DriftEvent(step=9, heads=((0, 2),), replace_fraction=0.9),
              DriftEvent(step=14, heads=((1, 5),), replace_fraction=0.8))
    return SynthSpec(num_layers=2, heads_per_layer=8, prefill_len=160, decode_steps=32,
                     trace_topk=48, archetypes=arch, clusters=clusters, drift_events=events,
                     seed=seed, bytes_per_kv_entry=512)


def taxonomy_json(tax):
    return {
        "roles": {hid(h): p.role for h, p in tax.heads.items()},
        "s_stable": {hid(h): p.s_stable for h, p in tax.heads.items()},
        "s_sim": {hid(h): p.s_sim for h, p in tax.heads.items()},
        "clusters": [[list(c.pivot), [list(s) for s in c.satellites]] for c in tax.clusters],
    }


def plan_json(plan):
    return {
        "rho": plan.rho, "prefill_len": plan.prefill_len, "num_heads": plan.num_heads,
        "num_full": plan.num_full, "num_comp": plan.num_comp, "l_base": plan.l_base,
        "l_base_int": plan.l_base_int,
        "lengths": {hid(h): n for h, n in plan.lengths.items()},
    }


def run_json(run):
    rep = run.report
    return {
        "rows": [r.to_json_dict() for r in rep.rows],
        "events": [e.to_json_dict() for e in rep.events],
        "final_gpu": {hid(h): sorted(s) for h, s in run.final_gpu.items()},
        "dynamic": {hid(h): sorted(s) for h, s in run.state.dynamic.items()},
        "trace_sha256": rep.trace_sha256,
        "aggregates": rep.aggregates(),
    }


def cfg_json(cfg):
    return {k: getattr(cfg, k) for k in (
        "tau_drift", "window", "transfer_bandwidth", "update_delay_steps", "sink_count",
        "recency_window", "variant", "eval_every_step")}


def dense_trace(seed, *, L=96, T=24, H=4, levels=6):
    """Dense rows (every position recorded) with heavy score ties and zeros,
    in the shape tensor mode produces; trace_topk = L + T."""
    rng = np.random.default_rng(seed)
    K = L + T
    idx = np.full((T + 1, 1, H, K), PAD_INDEX, dtype=np.uint32)
    sc = np.zeros((T + 1, 1, H, K), dtype=np.float32)
    hot = rng.permutation(L)[:L // 3]
    for s in range(T + 1):
        if s == T // 2:
            hot = rng.permutation(L)[:L // 3]
        n = L + s
        for h in range(H):
            w = (rng.integers(0, levels, size=n) / levels).astype(np.float32)
            w[hot[hot < n]] += np.float32(1.0 + (h % 2) * 0.5)
            w[rng.random(n) < 0.2] = 0.0
            order = np.lexsort((np.arange(n), -w.astype(np.float64)))
            idx[s, 0, h, :n] = order
            sc[s, 0, h, :n] = w[order]
    manifest = TraceManifest(model_name="dense", num_layers=1, heads_per_layer=H,
                             prefill_len=L, decode_steps=T, trace_topk=K,
                             pool_kernel_used=0, bytes_per_kv_entry=512)
    return make_trace(manifest, idx, sc)


def manual_taxonomy(roles, clusters, H, NL=1):
    heads = {}
    cid_of = {}
    for i, (p, sats) in enumerate(clusters):
        for m in (p, *sats):
            cid_of[m] = i
    for (l, h), r in roles.items():
        heads[(l, h)] = HeadProfile(layer=l, head=h, s_stable=0.3 + 0.1 * h if r in ("anchor", "satellite") else 0.2,
                                    s_sim=0.0, role=r, cluster_id=cid_of.get((l, h)))
    return TaxonomyResult(num_layers=NL, heads_per_layer=H, tau_stable=0.5, tau_sim=0.5,
                          profiling_topk=None, heads=heads,
                          clusters=tuple(Cluster(i, p, tuple(s)) for i, (p, s) in enumerate(clusters)))


def engine_cases():
    cases, arrays = [], {}

    def add(name, trace, tax, plan, cfg):
        run = CacheEngine(trace, tax, plan, cfg).run()
        m = trace.manifest
        arrays[name + "/indices"] = trace.indices
        arrays[name + "/scores"] = trace.scores
        cases.append({
            "name": name,
            "manifest": m.to_json_dict(),
            "taxonomy": taxonomy_json(tax),
            "plan": plan_json(plan),
            "config": cfg_json(cfg),
            "expected": run_json(run),
        })

    demo = json.loads((REF / "tests/data/demo_config.json").read_text())
    trace, _ = generate_synthetic(synth_spec_from_json(demo["synthetic"]))
    tax = run_taxonomy([trace], ProfileConfig(profiling_topk=24))
    plan = plan_budget(tax, BudgetConfig(rho=0.6, min_length=8), 400)
    add("demo", trace, tax, plan, EngineConfig(tau_drift=0.5, window=8, update_delay_steps=1))
    add("demo_no_retrieval", trace, tax, plan, EngineConfig(variant="no_retrieval"))

    def drift(name, cfg=EngineConfig(), **kw):
        tr, _ = generate_synthetic(drift_spec(**kw))
        tx = run_taxonomy([tr], ProfileConfig(profiling_topk=24))
        pl = plan_budget(tx, BudgetConfig(rho=0.6, min_length=8), 400)
        add(name, tr, tx, pl, cfg)

    for seed in (5, 6, 7):
        drift(f"drift_seed{seed}", seed=seed)
    drift("drift_no_allocation", EngineConfig(variant="no_allocation"), seed=9)
    drift("drift_no_retrieval", EngineConfig(variant="no_retrieval"), seed=9)
    drift("drift_delay3_bw500", EngineConfig(update_delay_steps=3, transfer_bandwidth=500), seed=11)
    for t0 in (17, 21, 24):
        drift(f"drift_t0_{t0}", seed=13, drift_step=t0)
    drift("drift_stable", seed=15, drift_step=None)
    drift("drift_sliding", EngineConfig(eval_every_step=True), seed=5)
    drift("drift_T64", seed=5, decode_steps=64)
    drift("drift_delay3", EngineConfig(update_delay_steps=3), seed=5)

    prof, bud = ProfileConfig(tau_sim=0.7), BudgetConfig(rho=0.5, min_length=6)
    for i in range(20):  # test_acceptance.py:173-210 replay suite
        rng = np.random.default_rng(7000 + i)
        L = int(rng.choice([40, 60, 80]))
        T = int(rng.choice([24, 32, 48]))
        agreement = float(rng.uniform(0.85, 0.95))
        shift = int(rng.integers(4, T - 3)) if i % 2 == 0 else None
        replace = float(rng.uniform(0.7, 0.9))
        spec = mixed_spec(int(rng.integers(0, 2**31)), prefill_len=L, decode_steps=T,
                          shift_step=shift, replace=replace, agreement=agreement)
        tr, _ = generate_synthetic(spec)
        tx = run_taxonomy([tr], prof)
        pl = plan_budget(tx, bud, L)
        cfg = EngineConfig(
            tau_drift=0.5, window=int(rng.choice([4, 8])),
            update_delay_steps=int(rng.choice([1, 2, 3])),
            transfer_bandwidth=int(rng.choice([300, 1 << 30])),
            variant=("heterocache", "no_allocation", "no_retrieval")[i % 3])
        add(f"replay_{i:02d}", tr, tx, pl, cfg)

    for seed in (21, 22):
        tr, _ = generate_synthetic(multi_layer_spec(seed))
        tx = run_taxonomy([tr], ProfileConfig(profiling_topk=16, tau_sim=0.6))
        pl = plan_budget(tx, BudgetConfig(rho=0.5, min_length=8), 160)
        add(f"multilayer_{seed}", tr, tx, pl, EngineConfig(window=4, update_delay_steps=2,
                                                            transfer_bandwidth=20000))

    roles = {(0, 0): "pivot", (0, 1): "satellite", (0, 2): "satellite", (0, 3): "anchor"}
    clusters = [((0, 0), ((0, 1), (0, 2)))]
    for seed in (31, 32, 33):
        tr = dense_trace(seed)
        tx = manual_taxonomy(roles, clusters, 4)
        pl = plan_budget(tx, BudgetConfig(rho=0.55, min_length=8), tr.manifest.prefill_len)
        add(f"dense_{seed}", tr, tx, pl, EngineConfig(window=4, update_delay_steps=1,
                                                       tau_drift=0.6, sink_count=4,
                                                       recency_window=8))
    return cases, arrays


def topk_cases():
    rng = np.random.default_rng(1234)
    out = []
    for n in (1, 2, 7, 40, 257, 1000, 2049):
        for trial in range(3):
            levels = int(rng.integers(2, 9))
            w = (rng.integers(0, levels, size=n) / levels).astype(np.float32)
            if trial == 2:
                w = (np.float32(0.9) ** np.arange(n, dtype=np.float32)).astype(np.float32)
                w = w[rng.permutation(n)]
            for k in sorted({1, max(1, n // 3), n, n + 3}):
                out.append({"kind": "dense", "w": w.tolist(), "k": k, "pool": 0,
                            "expected": sorted(top_k_indices(w.astype(np.float64), k))})
            for pool in (3, 5, 13):
                if pool > n:  # np.convolve 'same' returns max(n, pool) values
                    continue
                k = max(1, n // 4)
                out.append({"kind": "dense", "w": w.tolist(), "k": k, "pool": pool,
                            "expected": sorted(top_k_indices(w.astype(np.float64), k, pool_kernel=pool))})
            # sparse: a recorded top-K prefix with pads, scores nonincreasing
            K = min(n, 64)
            sel = rng.choice(max(n, K) + 50, size=K, replace=False)
            s = np.sort(w[:K])[::-1].astype(np.float32)
            live = int(rng.integers(1, K + 1))
            idx = np.full(K + 5, PAD_INDEX, dtype=np.uint32)
            sc = np.zeros(K + 5, dtype=np.float32)
            idx[:live] = sel[:live]
            sc[:live] = s[:live]
            pairs = list(zip(idx.tolist(), sc.tolist()))
            for k in sorted({1, max(1, live // 2), live, K + 5}):
                out.append({"kind": "sparse", "idx": idx.tolist(), "scores": sc.tolist(), "k": k,
                            "expected": sorted(top_k_indices(pairs, k))})
    return out


def budget_cases():
    rng = np.random.default_rng(99)
    out = []
    for i in range(120):
        n = int(rng.integers(1, 24))
        stab = {(0, j): float(rng.choice([rng.uniform(0, 1), 0.0, 1.0, 0.5])) for j in range(n)}
        L = int(rng.integers(16, 300000))
        l_base = float(rng.uniform(1.0, L * 0.8))
        cfg = BudgetConfig(rho=0.5, min_length=int(rng.choice([0, 8, 16, 64])),
                           rounding=("largest_remainder", "floor")[i % 5 == 4])
        try:
            plan = allocate(stab, l_base, cfg, prefill_len=L, num_full=int(rng.integers(0, 8)))
            exp = plan_json(plan)
        except Exception as exc:  # noqa: BLE001
            exp = {"error": type(exc).__name__}
        out.append({"stabilities": {hid(h): s for h, s in stab.items()}, "l_base": l_base,
                    "prefill_len": L, "num_full": None if "error" in exp else exp["num_full"],
                    "config": {"rho": 0.5, "min_length": cfg.min_length, "rounding": cfg.rounding,
                               "epsilon": cfg.epsilon},
                    "expected": exp})
    # the frozen allocation of test_budget.py:62-69 and the paper configs
    for rho, NL, pattern, L in ((0.325, 32, "llama", 229376), (0.2875, 28, "qwen", 131072),
                                (0.325, 32, "llama", 32768), (0.325, 1, "llama", 4096),
                                (0.325, 32, "llama", 65536)):
        per = (["pivot"] + ["satellite"] * 4 + ["anchor"] * 2 + ["volatile"]) if pattern == "llama" \
            else (["pivot"] + ["satellite"] * 2 + ["anchor"])
        roles = {(l, h): r for l in range(NL) for h, r in enumerate(per)}
        rng2 = np.random.default_rng(L + NL)
        heads = {hd: HeadProfile(layer=hd[0], head=hd[1], s_stable=float(rng2.uniform(0.2, 0.9)),
                                 s_sim=0.0, role=r, cluster_id=None if r in ("anchor", "volatile") else hd[0])
                 for hd, r in roles.items()}
        clusters = tuple(Cluster(l, (l, 0), tuple((l, h) for h in range(1, len(per)) if per[h] == "satellite"))
                         for l in range(NL))
        tax = TaxonomyResult(num_layers=NL, heads_per_layer=len(per), tau_stable=0.5, tau_sim=0.5,
                             profiling_topk=None, heads=heads, clusters=clusters)
        plan = plan_budget(tax, BudgetConfig(rho=rho, min_length=16), L)
        out.append({"plan_budget": True, "roles": {hid(h): r for h, r in roles.items()},
                    "stabilities": {hid(h): p.s_stable for h, p in heads.items()},
                    "prefill_len": L, "config": {"rho": rho, "min_length": 16,
                                                 "rounding": "largest_remainder", "epsilon": 1e-6},
                    "expected": plan_json(plan)})
    return out


def taxonomy_cases(arrays):
    out = []
    specs = [("demo_tax", drift_spec(seed=5), ProfileConfig(profiling_topk=24)),
             ("multi_tax", multi_layer_spec(21), ProfileConfig(profiling_topk=16, tau_sim=0.6))]
    for i in range(3):
        specs.append((f"mixed_tax_{i}", mixed_spec(4000 + i), ProfileConfig(tau_sim=0.7)))
    for name, spec, prof in specs:
        tr, _ = generate_synthetic(spec)
        tax = run_taxonomy([tr], prof)
        arrays[name + "/indices"] = tr.indices
        arrays[name + "/scores"] = tr.scores
        out.append({"name": name, "prefill_len": tr.manifest.prefill_len,
                    "config": {"tau_stable": prof.tau_stable, "tau_sim": prof.tau_sim,
                               "profiling_topk": prof.profiling_topk},
                    "expected": taxonomy_json(tax)})
    # multi-trace calibration (profiling.py:286-367: medians per trace, mean over traces;
    # SURVEY 8f rank 4): several traces of one geometry
    for name, seeds, prof in (("calib3", (4100, 4101, 4102), ProfileConfig(tau_sim=0.7)),
                              ("calib5", (4200, 4201, 4202, 4203, 4204),
                               ProfileConfig(tau_sim=0.6, profiling_topk=12))):
        trs = [generate_synthetic(mixed_spec(sd))[0] for sd in seeds]
        tax = run_taxonomy(trs, prof)
        names = []
        for i, tr in enumerate(trs):
            arrays[f"{name}/t{i}/indices"] = tr.indices
            arrays[f"{name}/t{i}/scores"] = tr.scores
            names.append(f"{name}/t{i}")
        out.append({"name": name, "traces": names, "prefill_len": trs[0].manifest.prefill_len,
                    "config": {"tau_stable": prof.tau_stable, "tau_sim": prof.tau_sim,
                               "profiling_topk": prof.profiling_topk},
                    "expected": taxonomy_json(tax)})
    return out


POLICY_TRACES = ("demo", "drift_seed5", "drift_t0_21", "replay_00", "replay_01", "replay_05",
                 "multilayer_21", "dense_31", "dense_32")


def policy_cases(cases, arrays):
    """run_policy (evaluation.py:165-228) for the baseline policies over engine-case traces."""
    from heterocache.trace import TraceManifest

    out = []
    for c in cases:
        if c["name"] not in POLICY_TRACES:
            continue
        m = TraceManifest(**c["manifest"])
        tr = make_trace(m, arrays[c["name"] + "/indices"], arrays[c["name"] + "/scores"])
        specs = [
            (PolicySpec("full_oracle"), None),
            (PolicySpec("static_topk", rho=0.1), None),
            (PolicySpec("static_topk", rho=0.35), EngineConfig(sink_count=8, recency_window=16)),
            (PolicySpec("static_topk", rho=0.6), EngineConfig(sink_count=0, recency_window=0)),
            (PolicySpec("sink_window", rho=0.3), None),
            (PolicySpec("sink_window", rho=0.5, sink_count=2, window=10), None),
            (PolicySpec("sink_window", rho=0.25, sink_count=0), None),
            (PolicySpec("static_topk", rho=0.01), None),   # k = floor(rho L) < 1 on short L
            (PolicySpec("sink_window", rho=0.05), None),   # sinks exceed floor(rho L)
        ]
        for spec, ecfg in specs:
            try:
                rep_ = run_policy(tr, spec, engine_config=ecfg)
                expected = rep_.to_json_dict()
            except Exception as exc:  # noqa: BLE001 -- record the reference's refusal
                expected = {"error": type(exc).__name__}
            out.append({"trace": c["name"], "policy": spec.name, "rho": spec.rho,
                        "sink_count": spec.sink_count, "window": spec.window,
                        "engine": None if ecfg is None else cfg_json(ecfg),
                        "expected": expected})
    return out


def main():
    cases, arrays = engine_cases()
    (OUT / "policy_cases.json").write_text(json.dumps(policy_cases(cases, arrays)))
    tax = taxonomy_cases(arrays)
    np.savez_compressed(OUT / "engine_traces.npz", **arrays)
    (OUT / "engine_cases.json").write_text(json.dumps(cases))
    (OUT / "taxonomy_cases.json").write_text(json.dumps(tax))
    (OUT / "topk_cases.json").write_text(json.dumps(topk_cases()))
    (OUT / "budget_cases.json").write_text(json.dumps(budget_cases()))
    shutil.copyfile(REF / "tests/data/golden_replay.json", OUT / "golden_replay.json")
    shutil.copyfile(REF / "tests/data/demo_config.json", OUT / "demo_config.json")
    for p in sorted(OUT.iterdir()):
        print(p.name, os.path.getsize(p))


if __name__ == "__main__":
    main()
