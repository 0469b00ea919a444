"""Pin the CPU oracle to the reference's own outputs (CPU only).

Every expectation here was produced by running the reference package
(tests/golden/make_golden.py); the oracle must reproduce it exactly before
it is trusted as the checker for the CUDA path.
"""

import math

import numpy as np
import pytest

from golden_io import case_inputs, engine_cases, expected_events, json_fixture, key, taxonomy_arrays
from oracle import hc_oracle as O

CASES = engine_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_replay_matches_reference(case):
    idx, sc, kw = case_inputs(case)
    got = O.replay(idx, sc, **kw)
    exp = case["expected"]
    assert len(got["rows"]) == len(exp["rows"])
    for g, e in zip(got["rows"], exp["rows"]):
        assert g["recall"] == pytest.approx(e["recall"], abs=1e-12)
        for f in ("gpu_entries", "extra_entries", "bytes_in_flight", "cumulative_bytes",
                  "retrieval_flag"):
            assert g[f] == e[f], (f, g["step"])
    assert got["events"] == expected_events(case)
    fin = {key(h): frozenset(v) for h, v in exp["final_gpu"].items()}
    assert got["final_gpu"] == fin
    dyn = {key(h): frozenset(v) for h, v in exp["dynamic"].items()}
    assert {h: frozenset(v) for h, v in got["dynamic"].items()} == dyn


def test_oracle_matches_reference_golden_replay_file():
    """pkg/tests/data/golden_replay.json (the reference's own golden)."""
    gold = json_fixture("golden_replay.json")
    case = next(c for c in CASES if c["name"] == "demo")
    idx, sc, kw = case_inputs(case)
    assert kw["l_base_int"] == gold["l_base_int"]
    assert {f"{h[0]},{h[1]}": n for h, n in kw["lengths"].items()} == gold["lengths"]
    got = O.replay(idx, sc, **kw)
    assert [r["gpu_entries"] for r in got["rows"]] == gold["charged"]
    assert [r["cumulative_bytes"] for r in got["rows"]] == gold["cumulative_bytes"]
    # recall: 1-ULP platform sensitivity of Python's sum()
    for a, b in zip([r["recall"] for r in got["rows"]], gold["recalls"]):
        assert a == pytest.approx(b, abs=1e-15)
    assert len(got["events"]) == len(gold["events"])
    for g, e in zip(got["events"], gold["events"]):
        assert g["trigger_step"] == e["trigger_step"]
        assert list(g["pivot"]) == list(e["pivot"])
        assert g["completion_step"] == e["completion_step"]
        assert g["transfer_bytes"] == e["transfer_bytes"]
        assert {f"{s[0]},{s[1]}": list(ix) for s, ix in g["fetches"]} == e["fetches"]


def test_oracle_topk_matches_reference():
    for c in json_fixture("topk_cases.json"):
        if c["kind"] == "dense":
            got = O.top_k_dense(np.asarray(c["w"], dtype=np.float32), c["k"], c["pool"])
        else:
            got = O.top_k_sparse(np.asarray(c["idx"], dtype=np.uint32),
                                 np.asarray(c["scores"], dtype=np.float32), c["k"])
        assert got.tolist() == c["expected"]


def test_oracle_budget_matches_reference():
    for c in json_fixture("budget_cases.json"):
        cfg = c["config"]
        exp = c["expected"]
        if c.get("plan_budget"):
            roles = {key(h): r for h, r in c["roles"].items()}
            stab = {key(h): s for h, s in c["stabilities"].items()}
            got = O.plan_budget(roles, stab, rho=cfg["rho"], prefill_len=c["prefill_len"],
                                epsilon=cfg["epsilon"], min_length=cfg["min_length"],
                                rounding=cfg["rounding"])
        else:
            stab = {key(h): s for h, s in c["stabilities"].items()}
            if "error" in exp:
                with pytest.raises(ValueError):
                    O.allocate(stab, c["l_base"], rho=cfg["rho"], epsilon=cfg["epsilon"],
                               min_length=cfg["min_length"], rounding=cfg["rounding"],
                               prefill_len=c["prefill_len"], num_full=0)
                continue
            got = O.allocate(stab, c["l_base"], rho=cfg["rho"], epsilon=cfg["epsilon"],
                             min_length=cfg["min_length"], rounding=cfg["rounding"],
                             prefill_len=c["prefill_len"], num_full=exp["num_full"])
        assert got["l_base"] == exp["l_base"]
        assert got["l_base_int"] == exp["l_base_int"]
        assert {f"{h[0]},{h[1]}": n for h, n in got["lengths"].items()} == exp["lengths"]


def test_oracle_taxonomy_matches_reference():
    for c in json_fixture("taxonomy_cases.json"):
        traces = [(*taxonomy_arrays(n), c["prefill_len"]) for n in c.get("traces", [c["name"]])]
        cfg = c["config"]
        roles, cluster_of, clusters, s_stable, s_sim = O.run_taxonomy(
            traces, tau_stable=cfg["tau_stable"], tau_sim=cfg["tau_sim"],
            profiling_topk=cfg["profiling_topk"])
        exp = c["expected"]
        assert {f"{h[0]},{h[1]}": r for h, r in roles.items()} == exp["roles"]
        assert [[list(p), [list(s) for s in sats]] for p, sats in clusters] == exp["clusters"]
        for h, v in exp["s_stable"].items():
            assert s_stable[key(h)] == v
            assert s_sim[key(h)] == exp["s_sim"][h]


def test_attention_oracle_semantics():
    torch = pytest.importorskip("torch")
    from oracle.attention_oracle import gqa_mean_row, unit_attention

    g = torch.Generator().manual_seed(0)
    q = torch.randn(4, 128, generator=g)
    k = torch.randn(50, 128, generator=g)
    v = torch.randn(50, 128, generator=g)
    o, p = unit_attention(q, k, v, [0, 3, 7, 9])
    s = (q @ k[[0, 3, 7, 9]].T) / math.sqrt(128)
    ref = torch.softmax(s.double(), -1)
    assert torch.allclose(p.double(), ref, atol=1e-6)
    assert torch.allclose(o.double(), ref @ v[[0, 3, 7, 9]].double(), atol=1e-5)
    row = gqa_mean_row(p)
    assert torch.allclose(row.double(), ref.mean(0), atol=1e-6)


def test_oracle_static_policies_match_reference_run_policy():
    """Baseline policies: the oracle's run_policy restatement
    reproduces the reference's reports (evaluation.py:165-228), refusals included."""
    from golden_io import case_arrays, engine_cases, policy_cases, policy_kwargs

    L = {c["name"]: c["manifest"]["prefill_len"] for c in engine_cases()}
    n = 0
    for pc in policy_cases():
        idx, sc = case_arrays(pc["trace"])
        kw = policy_kwargs(pc, L[pc["trace"]])
        exp = pc["expected"]
        if "error" in exp:
            with pytest.raises(O.PolicyError):
                O.static_policy_report(idx, sc, **kw)
            continue
        got = O.static_policy_report(idx, sc, **kw)
        assert got["rows"] == exp["rows"], (pc["trace"], pc["policy"], pc["rho"])
        assert got["budget_ceiling"] == exp["budget_ceiling"]
        assert got["update_delay_steps"] == exp["update_delay_steps"]
        assert got["events"] == list(exp["events"]) and got["policy"] == exp["policy"]
        n += 1
    assert n >= 50


def test_top_k_dense_select_matches_lexsort_order():
    """The O(n) selection the CPU decoder uses gives top_k_dense's exact output:
    random rows, rows with heavy ties at the k-th value, signed zeros, k at the
    edges, NaN rows (lexsort path)."""
    rng = np.random.default_rng(7)
    cases = []
    for n in (1, 2, 17, 1000, 4099):
        cases.append(rng.random(n, dtype=np.float32))
        cases.append(rng.integers(0, 5, n).astype(np.float32))  # few distinct values
        z = np.zeros(n, dtype=np.float32)
        z[::3] = -0.0
        z[::5] = 1.0
        cases.append(z)
        x = rng.random(n).astype(np.float32)
        x[rng.integers(0, n, max(1, n // 7))] = np.nan
        cases.append(x)
    for w in cases:
        n = w.size
        for k in sorted({0, 1, 2, n // 3, n // 2, n - 1, n, n + 3}):
            assert np.array_equal(O.top_k_dense_select(w, k), O.top_k_dense(w, k)), (n, k)
