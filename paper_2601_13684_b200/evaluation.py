"""Policy evaluation on the B200.

Mirror of the reference's ``heterocache.evaluation`` (evaluation.py:1-362):
the same ``PolicySpec``, ``run_policy``, ``run_policies``, ``compare`` and
errors, with every policy served by this package's GPU engines:

  full_oracle   every head keeps its whole cache (upper bound)      evaluation.py:192-196
  static_topk   per-head top-floor(rho L) of the step-0 record,
                engine sinks / recency tail, frozen for the decode   evaluation.py:198-214
  sink_window   sink_count sinks + a recency window of
                floor(rho L) - sink_count positions, no other entry  evaluation.py:216-228
  heterocache   role-aware plan with drift-triggered retrieval, and
                its variants no_allocation / no_retrieval            evaluation.py:230-253

A static policy is a fixed role assignment of the same engine: every head a
volatile (full) unit, or an anchor whose dynamic set is chosen once at
prefill and never refreshed.  Trace mode (``run_policy``) runs it through
the trace-driven ``engine.CacheEngine`` (K1 selection, float64 recall on
the GPU) and returns the reference's report (``_static_rows`` semantics:
update_delay_steps 0, no events, the policy's budget ceiling).  Tensor mode
(``policy_decoder``) serves it over real K/V with the fused attention
kernel -- the apples-to-apples speed comparison of bench.py --policy.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from math import floor
from typing import Optional

from .budget import BudgetConfig, BudgetPlan, plan_budget
from .profiling import ProfileConfig, run_taxonomy, taxonomy_from_roles
from .reporting import SimulationReport

HETEROCACHE_VARIANTS = ("heterocache", "no_allocation", "no_retrieval")
POLICY_NAMES = ("full_oracle", "static_topk", "sink_window") + HETEROCACHE_VARIANTS
STATIC_POLICIES = ("full_oracle", "static_topk", "sink_window")


class EvaluationError(ValueError):
    """Bad policy parameters or incomparable runs (evaluation.py:33-34)."""


class BudgetMismatchError(EvaluationError):
    """Policies given different entry budgets must not be compared (evaluation.py:37-38)."""


@dataclass(frozen=True)
class PolicySpec:
    """A named policy with its budget parameters (evaluation.py:62-102)."""

    name: str
    rho: float = 0.5
    sink_count: int = 4
    window: Optional[int] = None

    def __post_init__(self):
        if self.name not in POLICY_NAMES:
            raise EvaluationError(
                f"unknown policy {self.name!r}; expected one of {POLICY_NAMES}")
        if self.name != "full_oracle" and not 0.0 < self.rho <= 1.0:
            raise EvaluationError(f"rho must be in (0, 1], got {self.rho}")
        if self.window is not None and self.window < 0:
            raise EvaluationError(f"window must be nonnegative, got {self.window}")

    def effective_window(self, prefill_len: int) -> int:
        if self.window is not None:
            return self.window
        w = floor(self.rho * prefill_len) - self.sink_count
        if w < 0:
            raise EvaluationError(
                f"sink_count {self.sink_count} exceeds the budget "
                f"floor(rho * L) = {floor(self.rho * prefill_len)}")
        return w

    def budget_ceiling(self, num_heads: int, prefill_len: int) -> float:
        if self.name == "full_oracle":
            return float(num_heads * prefill_len)
        if self.name == "sink_window":
            per_head = min(self.sink_count + self.effective_window(prefill_len), prefill_len)
            return float(num_heads * per_head)
        return self.rho * num_heads * prefill_len


def parse_policy(name: str, rho: float, sink_count: int = 4,
                 window: Optional[int] = None) -> PolicySpec:
    return PolicySpec(name=name, rho=rho, sink_count=sink_count, window=window)


def static_roles(policy: PolicySpec, num_layers: int, heads_per_layer: int, prefill_len: int,
                 engine_config=None):
    """(taxonomy, plan, engine config) serving a static policy on the engine.

    full_oracle: every head volatile.  static_topk: every head an anchor with
    l_h = floor(rho L) under the engine's sinks / recency window.
    sink_window: every head an anchor with an empty dynamic set under the
    policy's sinks and a recency window of effective_window(L) positions.
    """
    from .engine import EngineConfig

    cfg = engine_config or EngineConfig()
    heads = [(l, h) for l in range(num_layers) for h in range(heads_per_layer)]
    N, L = len(heads), prefill_len
    if policy.name == "full_oracle":
        roles = {hd: "volatile" for hd in heads}
        plan = BudgetPlan(rho=1.0, prefill_len=L, num_heads=N, num_full=N, num_comp=0,
                          l_base=float(L), l_base_int=L, lengths={})
        cfg = replace(cfg, sink_count=0, recency_window=0, variant="no_retrieval")
    elif policy.name == "static_topk":
        k = floor(policy.rho * L)
        if k < 1:
            raise EvaluationError(f"rho {policy.rho} leaves no budget for static_topk")
        roles = {hd: "anchor" for hd in heads}
        plan = BudgetPlan(rho=policy.rho, prefill_len=L, num_heads=N, num_full=0, num_comp=N,
                          l_base=float(k), l_base_int=k, lengths={hd: k for hd in heads})
        cfg = replace(cfg, variant="no_retrieval")
    elif policy.name == "sink_window":
        window = policy.effective_window(L)
        roles = {hd: "anchor" for hd in heads}
        plan = BudgetPlan(rho=policy.rho, prefill_len=L, num_heads=N, num_full=0, num_comp=N,
                          l_base=1.0, l_base_int=1, lengths={hd: 0 for hd in heads})
        cfg = replace(cfg, sink_count=policy.sink_count, recency_window=window,
                      variant="no_retrieval")
    else:
        raise EvaluationError(f"{policy.name} is not a static policy")
    tax = taxonomy_from_roles(roles, [], num_layers=num_layers, heads_per_layer=heads_per_layer)
    return tax, plan, cfg


def _static_report(policy: PolicySpec, report: SimulationReport) -> SimulationReport:
    """Re-label an engine report as run_policy's _static_rows report (evaluation.py:151-162)."""
    return SimulationReport(
        policy=policy.name, trace_sha256=report.trace_sha256, num_layers=report.num_layers,
        heads_per_layer=report.heads_per_layer, prefill_len=report.prefill_len,
        decode_steps=report.decode_steps,
        budget_ceiling=policy.budget_ceiling(report.num_layers * report.heads_per_layer,
                                             report.prefill_len),
        update_delay_steps=0, rows=report.rows, events=())


def run_policy(trace, policy: PolicySpec, *, taxonomy=None, plan=None, engine_config=None,
               profile_config: Optional[ProfileConfig] = None,
               budget_config: Optional[BudgetConfig] = None,
               calibration_traces=None) -> SimulationReport:
    """Replay one policy over one trace on the GPU (evaluation.py:165-253)."""
    from . import engine as engine_mod

    m = trace.manifest
    if policy.name in STATIC_POLICIES:
        tax, pl, cfg = static_roles(policy, m.num_layers, m.heads_per_layer, m.prefill_len,
                                    engine_config)
        run = engine_mod.CacheEngine(trace, tax, pl, cfg).run()
        return _static_report(policy, run.report)
    cfg = engine_config or engine_mod.EngineConfig()
    if policy.name != cfg.variant:
        cfg = replace(cfg, variant=policy.name)
    if taxonomy is None:
        calib = list(calibration_traces) if calibration_traces else [trace]
        taxonomy = run_taxonomy(calib, profile_config or ProfileConfig())
    if plan is None:
        bcfg = budget_config or BudgetConfig(rho=policy.rho)
        if bcfg.rho != policy.rho:
            raise EvaluationError(
                f"budget config rho {bcfg.rho} disagrees with policy rho {policy.rho}")
        plan = plan_budget(taxonomy, bcfg, m.prefill_len)
    return engine_mod.run_simulation(trace, taxonomy, plan, cfg).report


def run_policies(trace, policies, **kwargs) -> list:
    """Run several policies on one trace, enforcing comparable budgets (evaluation.py:256-277)."""
    specs = list(policies)
    m = trace.manifest
    num_heads = m.num_layers * m.heads_per_layer
    ceilings = {s.name: s.budget_ceiling(num_heads, m.prefill_len)
                for s in specs if s.name != "full_oracle"}
    if ceilings:
        values = sorted(ceilings.values())
        if values[-1] - values[0] > num_heads + 1e-6:
            raise BudgetMismatchError(f"policy budgets differ beyond rounding slack: {ceilings}")
    return [run_policy(trace, s, **kwargs) for s in specs]


def compare(reports) -> dict:
    """One comparison table over reports of the same trace (evaluation.py:280-335)."""
    reports = list(reports)
    if not reports:
        raise EvaluationError("nothing to compare")
    names = [r.policy for r in reports]
    if len(set(names)) != len(names):
        raise EvaluationError(f"duplicate policy names: {names}")
    sha = {r.trace_sha256 for r in reports}
    if len(sha) != 1:
        raise EvaluationError("reports come from different traces")
    budgeted = [r for r in reports if r.policy != "full_oracle"]
    if budgeted:
        num_heads = budgeted[0].num_layers * budgeted[0].heads_per_layer
        ceilings = sorted(r.budget_ceiling for r in budgeted)
        if ceilings[-1] - ceilings[0] > num_heads + 1e-6:
            raise BudgetMismatchError(
                "reports use different entry budgets: "
                + ", ".join(f"{r.policy}={r.budget_ceiling}" for r in budgeted))
    table = []
    for r in sorted(reports, key=lambda r: r.policy):
        agg = r.aggregates()
        table.append({"policy": r.policy, "mean_recall": agg["mean_recall"],
                      "min_recall": agg["min_recall"],
                      "peak_gpu_entries": agg["peak_gpu_entries"],
                      "total_transfer_bytes": agg["total_transfer_bytes"],
                      "retrieval_events": agg["retrieval_events"],
                      "exposed_transfer_steps": agg["exposed_transfer_steps"],
                      "budget_ceiling": r.budget_ceiling})
    base = {row["policy"]: row["mean_recall"] for row in table}
    deltas = {n: base["heterocache"] - v for n, v in base.items()
              if "heterocache" in base and n != "heterocache"}
    return {"trace_sha256": sha.pop(), "policies": table,
            "mean_recall_delta_vs_heterocache": deltas}


def comparison_csv(comparison: dict) -> str:
    import csv
    import io

    columns = ("policy", "mean_recall", "min_recall", "peak_gpu_entries",
               "total_transfer_bytes", "retrieval_events", "exposed_transfer_steps",
               "budget_ceiling")
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(columns)
    for row in comparison["policies"]:
        w.writerow([row[c] for c in columns])
    return buf.getvalue()


# ---- tensor mode ------------------------------------------------------------


def policy_decoder(policy: PolicySpec, *, num_layers: int, heads_per_layer: int,
                   prefill_len: int, engine_config=None, taxonomy=None, plan=None,
                   **decoder_kw):
    """A HeteroCacheDecoder serving `policy` over real K/V (bench --policy).

    Static policies get their fixed role assignment (static_roles); the
    heterocache family needs its taxonomy and plan."""
    from .decoder import HeteroCacheDecoder
    from .engine import EngineConfig

    if policy.name in STATIC_POLICIES:
        taxonomy, plan, cfg = static_roles(policy, num_layers, heads_per_layer, prefill_len,
                                           engine_config)
    else:
        if taxonomy is None or plan is None:
            raise EvaluationError(f"{policy.name} needs a taxonomy and a plan")
        cfg = replace(engine_config or EngineConfig(), variant=policy.name)
    dec = HeteroCacheDecoder(taxonomy, plan, cfg, **decoder_kw)
    dec.policy = policy
    return dec


def policy_report(dec, b: int, decode_steps: int, trace_sha256: str = "") -> SimulationReport:
    """Report of sequence b of a policy decoder, labelled like run_policy's."""
    rep = dec.report(b, decode_steps, trace_sha256)
    policy = getattr(dec, "policy", None)
    if policy is not None and policy.name in STATIC_POLICIES:
        return _static_report(policy, rep)
    return rep
