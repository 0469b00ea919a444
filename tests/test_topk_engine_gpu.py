"""GPU parity: K1 selection, K2 overlap/drift and the trace-driven engine.

Bit-exact against (a) the reference's own outputs (golden fixtures produced
by tests/golden/make_golden.py) and (b) the pinned CPU oracle on larger,
tie-heavy rows.  Runs through the C ABI (libhcb200.so).
"""

import numpy as np
import pytest

from golden_io import case_arrays, engine_cases, expected_events, json_fixture, key, taxonomy_arrays
from oracle import hc_oracle as O

pytestmark = pytest.mark.gpu

CASES = engine_cases()


def _objects(case):
    from paper_2601_13684_b200.budget import BudgetPlan
    from paper_2601_13684_b200.engine import EngineConfig
    from paper_2601_13684_b200.profiling import taxonomy_from_roles
    from paper_2601_13684_b200.trace import TraceManifest, make_trace

    idx, sc = case_arrays(case["name"])
    m = TraceManifest(**case["manifest"])
    trace = make_trace(m, idx, sc)
    tx = case["taxonomy"]
    roles = {key(h): r for h, r in tx["roles"].items()}
    clusters = [(tuple(p), [tuple(s) for s in sats]) for p, sats in tx["clusters"]]
    tax = taxonomy_from_roles(roles, clusters, num_layers=m.num_layers,
                              heads_per_layer=m.heads_per_layer,
                              s_stable={key(h): v for h, v in tx["s_stable"].items()})
    p = case["plan"]
    plan = BudgetPlan(rho=p["rho"], prefill_len=p["prefill_len"], num_heads=p["num_heads"],
                      num_full=p["num_full"], num_comp=p["num_comp"], l_base=p["l_base"],
                      l_base_int=p["l_base_int"],
                      lengths={key(h): n for h, n in p["lengths"].items()})
    return trace, tax, plan, EngineConfig(**case["config"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_trace_engine_matches_reference_run(case):
    from paper_2601_13684_b200.engine import run_simulation

    trace, tax, plan, cfg = _objects(case)
    run = run_simulation(trace, tax, plan, cfg)
    exp = case["expected"]
    rows = [r.to_json_dict() for r in run.report.rows]
    assert len(rows) == len(exp["rows"])
    for g, e in zip(rows, exp["rows"]):
        # float64 record-order sums on device: identical bits to the reference run here
        assert g["recall"] == e["recall"], g["step"]
        assert g == e
    events = [dict(trigger_step=e.trigger_step, pivot=e.pivot, completion_step=e.completion_step,
                   transfer_bytes=e.transfer_bytes, fetches=e.fetches) for e in run.report.events]
    assert events == expected_events(case)
    assert {f"{h[0]},{h[1]}": sorted(v) for h, v in run.final_gpu.items()} == exp["final_gpu"]
    assert run.report.trace_sha256 == exp["trace_sha256"]
    assert run.report.aggregates() == exp["aggregates"]


def test_satellites_serve_stale_until_completion():
    """test_engine.py:164-184 against the GPU engine."""
    from paper_2601_13684_b200.engine import CacheEngine, EngineConfig

    case = next(c for c in CASES if c["name"] == "drift_delay3")
    trace, tax, plan, _ = _objects(case)
    eng = CacheEngine(trace, tax, plan, EngineConfig(update_delay_steps=3))
    state = eng.prefill_init()
    sat = (0, 2)
    initial = state.dynamic[sat]
    rows = {}
    for t in range(1, trace.manifest.decode_steps + 1):
        rows[t] = eng.decode_step(state, t)
        if t in (24, 25, 26):
            assert state.dynamic[sat] == initial
        if t == 27:
            assert state.dynamic[sat] != initial
    ev = state.events[0]
    assert (ev.trigger_step, ev.completion_step) == (24, 27)
    assert rows[24].bytes_in_flight == ev.transfer_bytes and rows[27].bytes_in_flight == 0


def test_topk_matches_reference_known_answers():
    from paper_2601_13684_b200.ops import topk_rows

    for c in json_fixture("topk_cases.json"):
        if c["kind"] == "dense":
            if c["pool"]:
                continue
            w = np.asarray(c["w"], dtype=np.float32)[None, :]
            sel, cnt = topk_rows(None, w, c["k"])
        else:
            sel, cnt = topk_rows(np.asarray(c["idx"], dtype=np.uint32)[None, :],
                                 np.asarray(c["scores"], dtype=np.float32)[None, :], c["k"])
        assert sorted(sel[0, :cnt[0]].tolist()) == c["expected"]


def test_pooled_dense_topk_matches_reference():
    """top_k_indices(dense, k, pool_kernel) on the GPU (hc_pooled_topk): the
    reference's known answers, then larger rows with ties and zeros against the
    oracle (np.convolve + lexsort, metrics.py:26-39)."""
    from paper_2601_13684_b200.ops import top_k_indices

    n = 0
    for c in json_fixture("topk_cases.json"):
        if c["kind"] == "dense" and c["pool"]:
            w = np.asarray(c["w"], dtype=np.float64)
            assert sorted(top_k_indices(w, c["k"], pool_kernel=c["pool"])) == c["expected"]
            n += 1
    assert n >= 20
    rng = np.random.default_rng(77)
    for size, pool in ((20000, 13), (131072, 5), (4097, 3), (50000, 13)):
        w = rng.random(size)
        w[rng.choice(size, size // 10)] = 0.0               # zero runs: pooled ties
        w[: size // 50] = np.round(w[: size // 50] * 4) / 4  # quantised: raw ties
        w[5] = -0.0
        for k in (1, 37, size // 3):
            want = O.top_k_dense(w, k, pool_kernel=pool)
            assert top_k_indices(w, k, pool_kernel=pool) == frozenset(int(x) for x in want)
    with pytest.raises(ValueError):
        top_k_indices(np.ones(5), 2, pool_kernel=7)
    with pytest.raises(ValueError):
        top_k_indices(np.ones(50), 2, pool_kernel=4)


def test_top_k_indices_dropin():
    from paper_2601_13684_b200.ops import top_k_indices

    assert top_k_indices(np.array([4.0, 1.0, 3.0, 2.0]), 2) == frozenset({0, 2})
    assert top_k_indices([(7, 0.5), (3, 0.5), (9, 0.9)], 2) == frozenset({9, 3})
    assert top_k_indices([(7, 0.5), (3, 0.5), (9, 0.9)], 10) == frozenset({3, 7, 9})
    assert top_k_indices([(4, 0.9), (2, 0.5), (0xFFFFFFFF, 0.0)], 3) == frozenset({4, 2})
    assert top_k_indices([], 4) == frozenset() and top_k_indices(np.array([1.0]), 0) == frozenset()


def _tie_heavy_rows(rng, R, n):
    rows = np.empty((R, n), dtype=np.float32)
    for r in range(R):
        kind = r % 4
        if kind == 0:  # few levels: massive ties
            rows[r] = rng.integers(0, 5, n) / 4
        elif kind == 1:  # geometric 0.9^i shuffled: subnormals and exact zeros
            rows[r] = (np.float32(0.9) ** np.arange(n, dtype=np.float32))[rng.permutation(n)]
        elif kind == 2:  # softmax-like with zeros and -0.0
            x = rng.standard_normal(n).astype(np.float32)
            x[rng.random(n) < 0.3] = 0.0
            x[rng.random(n) < 0.1] = -0.0
            rows[r] = np.abs(x) * (rng.random(n) < 0.9)
        else:  # all equal
            rows[r] = 0.25
    return rows


@pytest.mark.parametrize("n", [1, 31, 1000, 4097, 65536 + 17, 237568])
def test_dense_topk_bit_exact_vs_oracle(n):
    from paper_2601_13684_b200.ops import topk_rows

    rng = np.random.default_rng(n)
    rows = _tie_heavy_rows(rng, 8, n)
    ks = [1, max(1, n // 10), n // 2 + 1, n, n + 5, 3, max(1, n - 1), 7]
    sel, cnt = topk_rows(None, rows, ks)
    for r in range(rows.shape[0]):
        exp = O.top_k_dense(rows[r], ks[r])
        got = sel[r, :cnt[r]]
        assert np.array_equal(got, exp), (r, ks[r])  # dense output is already ascending


def test_overlap_counts_vs_bitmap():
    from paper_2601_13684_b200.ops import topk_rows

    rng = np.random.default_rng(7)
    n, R = 50000, 6
    rows = _tie_heavy_rows(rng, R, n)
    words = (n + 31) // 32
    bms = np.zeros((R, words), dtype=np.uint32)
    bases = []
    for r in range(R):
        b = rng.choice(n, size=n // 7, replace=False)
        bases.append(set(b.tolist()))
        np.bitwise_or.at(bms[r], b >> 5, np.uint32(1) << (b & 31).astype(np.uint32))
    sel, cnt, ovl = topk_rows(None, rows, 5000, base_bitmaps=bms)
    for r in range(R):
        exp = set(O.top_k_dense(rows[r], 5000).tolist())
        assert int(ovl[r]) == len(exp & bases[r])


def test_profiling_matches_reference_taxonomy():
    from paper_2601_13684_b200.profiling import ProfileConfig, run_taxonomy
    from paper_2601_13684_b200.trace import TraceManifest, make_trace

    for c in json_fixture("taxonomy_cases.json"):
        traces = []
        for name in c.get("traces", [c["name"]]):  # multi-trace calibration cases
            idx, sc = taxonomy_arrays(name)
            T1, NL, H, K = idx.shape
            m = TraceManifest("t", NL, H, c["prefill_len"], T1 - 1, K, 0, 256)
            traces.append(make_trace(m, idx, sc))
        tax = run_taxonomy(traces, ProfileConfig(**c["config"]))
        exp = c["expected"]
        assert {f"{l},{h}": p.role for (l, h), p in tax.heads.items()} == exp["roles"]
        assert [[list(cl.pivot), [list(s) for s in cl.satellites]] for cl in tax.clusters] \
            == exp["clusters"]
        for h, v in exp["s_stable"].items():
            assert tax.heads[key(h)].s_stable == v
            assert tax.heads[key(h)].s_sim == exp["s_sim"][h]


@pytest.mark.parametrize("n,k", [(740, 70), (4097, 410), (131072 + 5, 6554), (237568, 22938),
                                 (50000, 49999), (3000, 3000)])
def test_monitor_threshold_and_overlap_bit_exact(n, k):
    """Fused monitor K1+K2 (smem candidates and the streaming fallback for
    tie-heavy rows whose threshold bucket overflows) vs the oracle."""
    from paper_2601_13684_b200.ops import monitor_rows

    rng = np.random.default_rng(n + k)
    rows = _tie_heavy_rows(rng, 6, n)
    rows[4] = rng.dirichlet(np.full(n, 0.05)).astype(np.float32)  # softmax-like, heavy tail
    words = (n + 31) // 32
    bms = np.zeros((6, words), dtype=np.uint32)
    bases = []
    for r in range(6):
        b = rng.choice(n, size=max(1, n // 9), replace=False)
        bases.append(set(b.tolist()))
        np.bitwise_or.at(bms[r], b >> 5, np.uint32(1) << (b & 31).astype(np.uint32))
    thr, ovl = monitor_rows(rows, k, bms)
    for r in range(6):
        top = O.top_k_dense(rows[r], k)
        assert int(ovl[r]) == len(set(top.tolist()) & bases[r]), r
        # the threshold reproduces exactly the selected set
        keys = _composite_keys(rows[r])
        assert np.array_equal(np.nonzero(keys >= thr[r])[0].astype(np.uint32), top), r


def _composite_keys(row):
    u = row.astype(np.float32).view(np.uint32).copy()
    u[u == 0x80000000] = 0
    neg = (u & 0x80000000) != 0
    k32 = np.where(neg, ~u, u | np.uint32(0x80000000)).astype(np.uint64)
    pos = np.arange(row.size, dtype=np.uint64)
    return (k32 << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - pos)


def test_gram_counts_exact():
    """K6 tcgen05 Gram of indicator sets == exact set intersections."""
    import torch

    from paper_2601_13684_b200 import _lib

    rng = np.random.default_rng(3)
    B, S, k, n = 3, 150, 400, 5000
    sel = np.zeros((B, S, k), dtype=np.uint32)
    cnt = rng.integers(1, k + 1, size=(B, S)).astype(np.uint32)
    sets = []
    for b in range(B):
        for s in range(S):
            ids = rng.choice(n, size=int(cnt[b, s]), replace=False)
            sel[b, s, :cnt[b, s]] = ids
            sets.append(set(ids.tolist()))
    rows_pad = 256
    gram = torch.zeros((B, rows_pad, rows_pad), device="cuda")
    d_sel = torch.from_numpy(sel.view(np.int32)).cuda()
    d_cnt = torch.from_numpy(cnt.view(np.int32)).cuda()
    _lib.check(_lib.load().hc_gram_from_sets(d_sel.data_ptr(), d_cnt.data_ptr(), B, S, k, n,
                                             gram.data_ptr(), _lib.stream_handle()))
    g = gram.cpu().numpy()
    for b in range(B):
        for i in range(0, S, 7):
            for j in range(0, S, 5):
                assert g[b, i, j] == len(sets[b * S + i] & sets[b * S + j]), (b, i, j)
