"""CPU-only checks of the host mirror and the C ABI library (no compute calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from golden_io import case_arrays, engine_cases, json_fixture, key

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    from paper_2601_13684_b200 import _lib

    lib = _lib.load()
    header = (ROOT / "include" / "hcb200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|const char\*|void|unsigned long long)\s+(hc_\w+)\s*\(",
                              header, re.M))
    assert declared, "no entry points parsed from include/hcb200.h"
    for name in sorted(declared):
        assert hasattr(lib, name), f"libhcb200.so does not export {name}"
    assert set(_lib.EXPORTED) == declared, "ctypes declarations out of sync with the header"
    assert lib.hc_version().startswith(b"hcb200")


def test_library_rejects_bad_arguments_without_gpu():
    from paper_2601_13684_b200 import _lib

    lib = _lib.load()
    assert lib.hc_topk_batched(None, 3, 0, None) == _lib.HC_EINVAL
    assert b"bad jobs" in lib.hc_last_error()


def test_budget_matches_reference_fixtures():
    from paper_2601_13684_b200.budget import BudgetConfig, BudgetError, allocate
    from paper_2601_13684_b200.profiling import taxonomy_from_roles
    from paper_2601_13684_b200.budget import plan_budget

    for c in json_fixture("budget_cases.json"):
        cfg = c["config"]
        exp = c["expected"]
        bc = BudgetConfig(rho=cfg["rho"], epsilon=cfg["epsilon"], min_length=cfg["min_length"],
                          rounding=cfg["rounding"])
        stab = {key(h): s for h, s in c["stabilities"].items()}
        if c.get("plan_budget"):
            roles = {key(h): r for h, r in c["roles"].items()}
            NL = 1 + max(l for l, _ in roles)
            H = 1 + max(h for _, h in roles)
            clusters = []
            for l in range(NL):
                sats = [(l, h) for h in range(H) if roles[(l, h)] == "satellite"]
                clusters.append(((l, 0), sats))
            tax = taxonomy_from_roles(roles, clusters, num_layers=NL, heads_per_layer=H,
                                      s_stable=stab)
            got = plan_budget(tax, bc, c["prefill_len"])
        elif "error" in exp:
            with pytest.raises(BudgetError):
                allocate(stab, c["l_base"], bc, prefill_len=c["prefill_len"], num_full=0)
            continue
        else:
            got = allocate(stab, c["l_base"], bc, prefill_len=c["prefill_len"],
                           num_full=exp["num_full"])
        assert got.l_base == exp["l_base"]
        assert got.l_base_int == exp["l_base_int"]
        assert {f"{l},{h}": n for (l, h), n in got.lengths.items()} == exp["lengths"]


def test_trace_roundtrip_and_fingerprint():
    from paper_2601_13684_b200.trace import (BadMagicError, TraceManifest,
                                             TruncatedPayloadError, make_trace, read_trace,
                                             trace_bytes, trace_fingerprint)

    for case in engine_cases()[:6]:
        idx, sc = case_arrays(case["name"])
        m = TraceManifest(**case["manifest"])
        tr = make_trace(m, idx, sc)
        assert trace_fingerprint(tr) == case["expected"]["trace_sha256"]
        blob = trace_bytes(tr)
        back = read_trace(blob)
        assert np.array_equal(back.indices, tr.indices) and np.array_equal(back.scores, tr.scores)
        with pytest.raises(BadMagicError):
            read_trace(b"NOTATRACE" + blob[9:])
        with pytest.raises(TruncatedPayloadError):
            read_trace(blob[:-3])


def test_engine_config_validation_and_cache_view():
    from paper_2601_13684_b200.engine import CacheView, EngineConfig, EngineError

    for bad in (dict(tau_drift=2.0), dict(window=0), dict(transfer_bandwidth=0),
                dict(update_delay_steps=-1), dict(variant="turbo")):
        with pytest.raises(EngineError):
            EngineConfig(**bad)
    view = CacheView(prefill_len=100, step=5, base=frozenset({50}), sink_count=4, recency_window=8)
    assert 50 in view and 0 in view and 3 in view and 4 not in view
    assert 97 in view and 96 not in view and 104 in view
    comp = CacheView(prefill_len=100, step=5, base=frozenset({0, 50}), sink_count=4,
                     recency_window=8)
    assert comp.size() == len({0, 50} | {0, 1, 2, 3} | {97, 98, 99}) + 5


def test_completion_step_rule():
    from paper_2601_13684_b200.engine import EngineConfig, completion_step

    cfg = EngineConfig(update_delay_steps=3, transfer_bandwidth=500)
    assert completion_step(24, 24576, cfg) == 50
    assert completion_step(24, 1000, cfg) == 27


def test_sass_proves_blackwell_native_kernels():
    """cuobjdump of libhcb200.so: tcgen05 MMAs (UTC*MMA), TMEM loads (LDTM),
    TMA tensor loads (UTMALDG) -- the sm_100a evidence of K5 / K4."""
    import shutil
    import subprocess

    from paper_2601_13684_b200 import _lib

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert re.search(r"UTC\w*MMA", out), "no tcgen05 MMA in the SASS"
    assert "LDTM" in out, "no tcgen05.ld (TMEM load) in the SASS"
    assert "UTMALDG" in out, "no TMA tensor load in the SASS"


def test_window_median_bit_identical_to_numpy():
    from paper_2601_13684_b200.decoder import window_median

    rng = np.random.default_rng(0)
    for W in (1, 2, 3, 4, 7, 8, 9, 16):
        for _ in range(50):
            v = rng.integers(0, 6555, size=(W, 37)) / 6554  # overlap counts / l_base_int
            v[rng.random(v.shape) < 0.3] = 0.5
            got = window_median(v)
            exp = np.median(v, axis=0)
            assert np.array_equal(got, exp)
            for j in range(v.shape[1]):  # the reference's per-list call (engine.py:250)
                assert got[j] == np.median(list(v[:, j]))


def test_policy_spec_mirrors_reference_rules():
    """evaluation.PolicySpec / run_policies / compare host logic (evaluation.py:62-335),
    checked against the oracle's restatement of the budget rules -- no GPU needed."""
    from paper_2601_13684_b200.evaluation import (BudgetMismatchError, EvaluationError,
                                                  PolicySpec, compare, comparison_csv,
                                                  static_roles)
    from paper_2601_13684_b200.reporting import SimulationReport, StepRow
    from oracle import hc_oracle as O

    with pytest.raises(EvaluationError):
        PolicySpec("lru")
    with pytest.raises(EvaluationError):
        PolicySpec("static_topk", rho=0.0)
    with pytest.raises(EvaluationError):
        PolicySpec("sink_window", window=-1)
    for name, rho, sinks, window, L in [("sink_window", 0.3, 4, None, 400),
                                        ("sink_window", 0.5, 2, 10, 60),
                                        ("static_topk", 0.35, 4, None, 96),
                                        ("full_oracle", 0.5, 4, None, 400)]:
        spec = PolicySpec(name, rho=rho, sink_count=sinks, window=window)
        assert spec.budget_ceiling(12, L) == O.policy_budget_ceiling(name, rho, sinks, window,
                                                                      12, L)
    with pytest.raises(EvaluationError):
        PolicySpec("sink_window", rho=0.05).effective_window(60)
    with pytest.raises(EvaluationError):
        static_roles(PolicySpec("static_topk", rho=0.01), 1, 4, 60)
    tax, plan, cfg = static_roles(PolicySpec("sink_window", rho=0.3), 2, 4, 400)
    assert set(tax.compressed_heads()) == set(plan.lengths) and not any(plan.lengths.values())
    assert (cfg.sink_count, cfg.recency_window, cfg.variant) == (4, 116, "no_retrieval")

    def rep(policy, recalls, ceiling, sha="x"):
        rows = tuple(StepRow(step=t, recall=r, gpu_entries=10, extra_entries=0,
                             bytes_in_flight=0, cumulative_bytes=0, retrieval_flag=0)
                     for t, r in enumerate(recalls))
        return SimulationReport(policy=policy, trace_sha256=sha, num_layers=1,
                                heads_per_layer=4, prefill_len=100, decode_steps=len(rows) - 1,
                                budget_ceiling=ceiling, update_delay_steps=0, rows=rows,
                                events=())

    table = compare([rep("static_topk", [1.0, 0.5], 40.0), rep("heterocache", [1.0, 0.9], 40.0),
                     rep("full_oracle", [1.0, 1.0], 400.0)])
    assert [r["policy"] for r in table["policies"]] == ["full_oracle", "heterocache",
                                                        "static_topk"]
    assert table["mean_recall_delta_vs_heterocache"]["static_topk"] == 0.95 - 0.75
    assert comparison_csv(table).splitlines()[0].startswith("policy,mean_recall")
    with pytest.raises(BudgetMismatchError):
        compare([rep("static_topk", [1.0], 40.0), rep("sink_window", [1.0], 80.0)])
    with pytest.raises(EvaluationError):
        compare([rep("static_topk", [1.0], 40.0), rep("heterocache", [1.0], 40.0, sha="y")])


def test_library_has_no_unresolved_internal_symbols():
    """Every hc:: function the translation units call is defined in the library
    (a missing definition would only surface as a dlopen failure on the GPU box)."""
    import shutil
    import subprocess

    from paper_2601_13684_b200 import _lib

    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--undefined-only", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    missing = [ln.split()[-1] for ln in out.splitlines() if "_ZN2hc" in ln]
    assert not missing, missing
