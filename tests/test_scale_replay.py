"""Parity closed at 128K context -- CPU only.

tests/golden/scale_128k/ holds an HCTRACE1-shaped export of a tensor-mode GPU
run in measure mode (tools/export_trace.py on a B200: Qwen2.5-7B-shaped,
131,072-token prefill, 2 layers, planted topic shift): every head's records
at every step (pivots: top-l_base_int of their own decision rows; the others:
top-1024 of their dense GPU rows), plus the GPU engine's event log, full
StepRows (recall computed on the GPU) and final dynamic
sets.  Replaying the trace through the REFERENCE engine
(heterocache.engine.CacheEngine, imported from /root/reference when it is
mounted) and through the pinned oracle must reproduce the GPU's decisions
and StepRows -- recall included -- exactly.
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from golden_io import key
from oracle import hc_oracle as O

DIR = Path(__file__).resolve().parent / "golden" / "scale_128k"
REF = Path("/root/reference/pkg")


def _load():
    run = json.loads((DIR / "scale_run.json").read_text())
    with np.load(DIR / "scale_trace.npz") as z:
        return run, z["indices"], z["scores"]


def _gpu_events(run):
    return [dict(trigger_step=e["trigger_step"], pivot=tuple(e["pivot"]),
                 completion_step=e["completion_step"], transfer_bytes=e["transfer_bytes"],
                 fetches=tuple((tuple(f["satellite"]), tuple(f["indices"])) for f in e["fetches"]))
            for e in run["gpu_events"]]


def test_oracle_replay_of_gpu_trace_at_128k():
    run, idx, sc = _load()
    cfg = run["config"]
    out = O.replay(idx, sc, prefill_len=run["manifest"]["prefill_len"],
                   bytes_per_kv_entry=run["manifest"]["bytes_per_kv_entry"],
                   roles={key(h): r for h, r in run["roles"].items()},
                   clusters=[(tuple(p), tuple(tuple(s) for s in sats)) for p, sats in run["clusters"]],
                   lengths={key(h): n for h, n in run["plan"]["lengths"].items()},
                   l_base_int=run["plan"]["l_base_int"], measure=True, **cfg)
    assert run["gpu_events"], "the planted shift must fire"
    assert out["events"] == _gpu_events(run)
    assert len(run["gpu_rows"]) == len(out["rows"])
    for g, e in zip(run["gpu_rows"], out["rows"]):
        assert g == e
    assert {f"{h[0]},{h[1]}": sorted(v) for h, v in out["dynamic"].items()} == run["gpu_dynamic"]


@pytest.mark.skipif(not REF.exists(), reason="reference package not mounted")
def test_reference_engine_replays_gpu_trace_at_128k():
    sys.path[:0] = [str(REF / "src")]
    try:
        from heterocache.budget import BudgetPlan
        from heterocache.engine import CacheEngine, EngineConfig
        from heterocache.profiling import Cluster, HeadProfile, TaxonomyResult
        from heterocache.trace import TraceManifest, make_trace
    finally:
        del sys.path[0]
    from heterocache.trace import read_trace as ref_read_trace

    from paper_2601_13684_b200 import trace as ours

    run, idx, sc = _load()
    # byte-level HCTRACE1 compatibility: written by this package, parsed by the reference
    blob = ours.trace_bytes(ours.make_trace(ours.TraceManifest(**run["manifest"]), idx, sc))
    trace = ref_read_trace(blob)
    assert trace.manifest == TraceManifest(**run["manifest"])
    cid = {}
    clusters = []
    for i, (p, sats) in enumerate(run["clusters"]):
        clusters.append(Cluster(i, tuple(p), tuple(tuple(s) for s in sats)))
        for m in [tuple(p)] + [tuple(s) for s in sats]:
            cid[m] = i
    heads = {key(h): HeadProfile(layer=key(h)[0], head=key(h)[1], s_stable=run["s_stable"][h],
                                 s_sim=0.0, role=r, cluster_id=cid.get(key(h)))
             for h, r in run["roles"].items()}
    m = run["manifest"]
    tax = TaxonomyResult(num_layers=m["num_layers"], heads_per_layer=m["heads_per_layer"],
                         tau_stable=0.5, tau_sim=0.5, profiling_topk=None, heads=heads,
                         clusters=tuple(clusters))
    p = run["plan"]
    plan = BudgetPlan(rho=p["rho"], prefill_len=p["prefill_len"], num_heads=p["num_heads"],
                      num_full=p["num_full"], num_comp=p["num_comp"], l_base=p["l_base"],
                      l_base_int=p["l_base_int"],
                      lengths={key(h): n for h, n in p["lengths"].items()})
    ref = CacheEngine(trace, tax, plan, EngineConfig(**run["config"])).run()
    got = [dict(trigger_step=e.trigger_step, pivot=e.pivot, completion_step=e.completion_step,
                transfer_bytes=e.transfer_bytes, fetches=e.fetches) for e in ref.report.events]
    assert got == _gpu_events(run)
    assert len(run["gpu_rows"]) == len(ref.report.rows)
    assert any(r["recall"] < 1.0 for r in run["gpu_rows"]), "compressed heads must miss some mass"
    for g, r in zip(run["gpu_rows"], ref.report.rows):
        assert g == r.to_json_dict()
    assert {f"{h[0]},{h[1]}": sorted(v) for h, v in ref.state.dynamic.items()} == run["gpu_dynamic"]
