"""Loaders for the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def key(s: str) -> tuple:
    a, b = s.split(",")
    return (int(a), int(b))


@lru_cache(maxsize=None)
def _traces():
    with np.load(GOLDEN / "engine_traces.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=None)
def engine_cases():
    return json.loads((GOLDEN / "engine_cases.json").read_text())


def case_arrays(name):
    t = _traces()
    return t[name + "/indices"], t[name + "/scores"]


def case_inputs(case):
    """(indices, scores, kwargs for oracle.replay / engine) from one case."""
    idx, sc = case_arrays(case["name"])
    tax = case["taxonomy"]
    roles = {key(h): r for h, r in tax["roles"].items()}
    clusters = [(tuple(p), tuple(tuple(s) for s in sats)) for p, sats in tax["clusters"]]
    plan = case["plan"]
    lengths = {key(h): n for h, n in plan["lengths"].items()}
    cfg = case["config"]
    kw = dict(prefill_len=case["manifest"]["prefill_len"],
              bytes_per_kv_entry=case["manifest"]["bytes_per_kv_entry"],
              roles=roles, clusters=clusters, lengths=lengths,
              l_base_int=plan["l_base_int"], tau_drift=cfg["tau_drift"], window=cfg["window"],
              transfer_bandwidth=cfg["transfer_bandwidth"],
              update_delay_steps=cfg["update_delay_steps"], sink_count=cfg["sink_count"],
              recency_window=cfg["recency_window"], variant=cfg["variant"],
              eval_every_step=cfg["eval_every_step"])
    return idx, sc, kw


def expected_events(case):
    out = []
    for e in case["expected"]["events"]:
        out.append(dict(trigger_step=e["trigger_step"], pivot=tuple(e["pivot"]),
                        completion_step=e["completion_step"],
                        transfer_bytes=e["transfer_bytes"],
                        fetches=tuple((tuple(f["satellite"]), tuple(f["indices"]))
                                      for f in e["fetches"])))
    return out


@lru_cache(maxsize=None)
def json_fixture(name):
    return json.loads((GOLDEN / name).read_text())


def taxonomy_arrays(name):
    t = _traces()
    return t[name + "/indices"], t[name + "/scores"]


@lru_cache(maxsize=None)
def policy_cases():
    return json.loads((GOLDEN / "policy_cases.json").read_text())


def policy_kwargs(pc, prefill_len):
    """kwargs of oracle.static_policy_report for one policy case."""
    eng = pc["engine"] or {"sink_count": 4, "recency_window": 8}  # EngineConfig() defaults
    return dict(prefill_len=prefill_len, name=pc["policy"], rho=pc["rho"],
                sink_count=pc["sink_count"], window=pc["window"],
                engine_sink_count=eng["sink_count"], engine_recency_window=eng["recency_window"])
