"""Drop-in CacheEngine whose per-step work runs on the B200.

Same constructor, methods, state object, errors and outputs as the
reference engine (engine.py:44-425): ``CacheEngine(trace, taxonomy, plan,
config)`` with ``prefill_init() -> CacheState``, ``decode_step(state, step)
-> StepRow`` and ``run() -> EngineRun``.  It accepts the reference's own
trace / taxonomy / plan objects or this package's (duck-typed).

What moves to the GPU (per decode step, one stream, one host sync):
  * K1 top-k of every pivot row with the |top & K_base| count fused in
    (pivot_top_set / pivot_overlap, engine.py:232-245, 305-311);
  * K1 fetch selection for every satellite of a firing pivot
    (engine.py:326-329) and prefill selections (engine.py:263-274);
  * per-head residency recall in float64 record order (_measure,
    engine.py:276-288), with dynamic sets held as device bitmaps.
What stays on the host, exactly as the reference writes it: landing order
of due transfers, the window median test (drift_check, engine.py:247-250),
byte accounting and completion steps (engine.py:330-347), event records.

This is the trace-driven mode used for bit-exact parity against the
reference simulator.  The tensor-mode decoder (decoder.py) runs the same
decision logic over real K/V and the fused attention kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil
from typing import Optional

import numpy as np

from . import _lib
from .ops import RECALL_HEAD_DTYPE, TOPK_JOB_DTYPE, launch_topk, to_device_struct
from .reporting import RetrievalRecord, SimulationReport, StepRow
from .trace import PAD_INDEX, trace_fingerprint

VARIANTS = ("heterocache", "no_allocation", "no_retrieval")


class EngineError(RuntimeError):
    """Inconsistent inputs (engine.py:44-45)."""


class InfeasibleStateError(EngineError):
    """The trace or budget cannot support the simulation (engine.py:48-49)."""


@dataclass(frozen=True)
class EngineConfig:
    tau_drift: float = 0.5
    window: int = 8
    transfer_bandwidth: int = 1 << 30
    update_delay_steps: int = 1
    sink_count: int = 4
    recency_window: int = 8
    variant: str = "heterocache"
    eval_every_step: bool = False

    def __post_init__(self):
        if not (0.0 <= self.tau_drift <= 1.0):
            raise EngineError(f"tau_drift must be in [0, 1], got {self.tau_drift}")
        if self.window < 1:
            raise EngineError(f"window must be positive, got {self.window}")
        if self.transfer_bandwidth < 1:
            raise EngineError(f"transfer_bandwidth must be positive, got {self.transfer_bandwidth}")
        if self.update_delay_steps < 0:
            raise EngineError(f"update_delay_steps must be nonnegative, got {self.update_delay_steps}")
        if self.sink_count < 0 or self.recency_window < 0:
            raise EngineError("sink_count and recency_window must be nonnegative")
        if self.variant not in VARIANTS:
            raise EngineError(f"unknown variant {self.variant!r}; expected {VARIANTS}")


@dataclass(frozen=True)
class CacheView:
    """Residency of one head at one step (engine.py:82-115)."""

    prefill_len: int
    step: int
    base: Optional[frozenset]
    sink_count: int
    recency_window: int

    def __contains__(self, position: int) -> bool:
        L = self.prefill_len
        if position >= L or self.base is None or position < self.sink_count:
            return True
        if position >= L + self.step - self.recency_window:
            return True
        return position in self.base

    def extras(self) -> set:
        L, t = self.prefill_len, self.step
        out = set(range(min(self.sink_count, L)))
        out.update(range(max(0, L + t - self.recency_window), L))
        return out

    def size(self) -> int:
        if self.base is None:
            return self.prefill_len + self.step
        # |base U extras| without materialising the union (base holds thousands of
        # positions, extras only sinks + the recency tail)
        extras = self.extras()
        return len(self.base) + sum(1 for x in extras if x not in self.base) + self.step


@dataclass
class _Transfer:
    completion_step: int
    order: int
    satellite: tuple
    indices: frozenset


@dataclass
class CacheState:
    step: int
    dynamic: dict
    k_base: dict
    buffers: dict
    buffer_steps: dict
    pending: list = field(default_factory=list)
    events: list = field(default_factory=list)
    cumulative_bytes: int = 0
    _order_counter: int = 0

    def bytes_in_flight(self, step: int) -> int:
        return sum(e.transfer_bytes for e in self.events if e.completion_step > step)


@dataclass(frozen=True)
class EngineRun:
    report: SimulationReport
    final_gpu: dict
    state: CacheState


def completion_step(step: int, cumulative_bytes: int, cfg: EngineConfig) -> int:
    """engine.py:334-337 (float true division then ceil, as in Python)."""
    return max(step + cfg.update_delay_steps, ceil(cumulative_bytes / cfg.transfer_bandwidth))


class CacheEngine:
    """Binds one trace to a taxonomy, a plan and the drift knobs; runs on the GPU."""

    def __init__(self, trace, taxonomy, plan, config: EngineConfig = EngineConfig()):
        m = trace.manifest
        if (taxonomy.num_layers, taxonomy.heads_per_layer) != (m.num_layers, m.heads_per_layer):
            raise EngineError(
                "taxonomy geometry does not match the trace: "
                f"{taxonomy.num_layers}x{taxonomy.heads_per_layer} vs "
                f"{m.num_layers}x{m.heads_per_layer}")
        if plan.prefill_len != m.prefill_len:
            raise EngineError(f"plan was made for prefill {plan.prefill_len}, trace has {m.prefill_len}")
        self.trace, self.taxonomy, self.plan, self.config = trace, taxonomy, plan, config
        self.heads = [(l, h) for l in range(m.num_layers) for h in range(m.heads_per_layer)]
        self.full = set(taxonomy.full_heads())
        self.comp = list(taxonomy.compressed_heads())
        if set(plan.lengths) != set(self.comp):
            raise EngineError("plan does not cover exactly the compressed heads")
        self.pivots = list(taxonomy.pivots())
        self.satellites_of = {p: tuple(taxonomy.cluster_of(p).satellites) for p in self.pivots}
        self.l_base_int = plan.l_base_int
        if self.l_base_int < 1:
            raise InfeasibleStateError(
                f"per-head base budget rounds to {self.l_base_int}; nothing to monitor")
        monitoring = bool(self.pivots) and config.variant != "no_retrieval"
        if monitoring and m.trace_topk < self.l_base_int:
            raise InfeasibleStateError(
                f"trace records only {m.trace_topk} entries per head but drift "
                f"monitoring needs the top {self.l_base_int}")
        planned = plan.num_full * m.prefill_len + (
            len(self.comp) * self.l_base_int if config.variant == "no_allocation"
            else sum(plan.lengths.values()))
        if planned > plan.budget_ceiling + plan.num_comp + 1e-9:
            raise InfeasibleStateError(
                f"planned GPU entries {planned} exceed the budget ceiling "
                f"{plan.budget_ceiling} plus rounding slack {plan.num_comp}")
        self._dev = None

    # ---- device residency -------------------------------------------------

    def _device(self):
        """Upload the trace once and lay out bitmaps / job templates."""
        if self._dev is not None:
            return self._dev
        import torch

        _lib.require_cuda()
        m = self.trace.manifest
        T1, NL, H, K = self.trace.indices.shape
        d = {}
        d["idx"] = torch.from_numpy(np.array(self.trace.indices, copy=True).view(np.int32)).cuda()
        d["sc"] = torch.from_numpy(np.array(self.trace.scores, copy=True)).cuda()
        d["K"] = K
        d["stride"] = NL * H * K  # elements per step record
        d["row"] = {hd: hd[0] * H + hd[1] for hd in self.heads}
        words = (m.prefill_len + m.decode_steps + 31) // 32 + 1
        d["words"] = words
        d["comp_slot"] = {hd: i for i, hd in enumerate(self.comp)}
        d["dyn_bm"] = torch.zeros((max(1, len(self.comp)), words), dtype=torch.int32, device="cuda")
        d["piv_slot"] = {p: i for i, p in enumerate(self.pivots)}
        npv = max(1, len(self.pivots))
        d["kbase_bm"] = torch.zeros((npv, words), dtype=torch.int32, device="cuda")
        kcap = max([self.l_base_int] + [self.effective_length(s) for p in self.pivots
                                        for s in self.satellites_of[p]] + [1])
        d["kcap"] = kcap
        d["top_idx"] = torch.zeros((npv, kcap), dtype=torch.int32, device="cuda")
        d["top_cnt"] = torch.zeros(npv, dtype=torch.int32, device="cuda")
        d["ovl"] = torch.zeros(npv, dtype=torch.int32, device="cuda")
        nh = len(self.heads)
        d["recall"] = torch.zeros(nh, dtype=torch.float64, device="cuda")
        rh = np.zeros(nh, dtype=RECALL_HEAD_DTYPE)
        for i, hd in enumerate(self.heads):
            off = d["row"][hd] * K * 4
            rh[i]["idx"] = _lib.ptr(d["idx"]) + off
            rh[i]["scores"] = _lib.ptr(d["sc"]) + off
            if hd not in self.full:
                rh[i]["dynamic"] = _lib.ptr(d["dyn_bm"]) + d["comp_slot"][hd] * words * 4
        d["recall_heads"] = to_device_struct(rh)
        self._dev = d
        return d

    def _row_ptrs(self, step: int, hd) -> tuple:
        d = self._device()
        off = (step * d["stride"] + d["row"][hd] * d["K"]) * 4
        return _lib.ptr(d["sc"]) + off, _lib.ptr(d["idx"]) + off

    def _select(self, requests):
        """Run K1 on [(step, head, k, out_idx_ptr, out_cnt_ptr, base_bm_ptr, ovl_ptr)]."""
        d = self._device()
        jobs = np.zeros(len(requests), dtype=TOPK_JOB_DTYPE)
        for i, (step, hd, k, oi, oc, bb, ov) in enumerate(requests):
            sp, ip = self._row_ptrs(step, hd)
            jobs[i] = (sp, ip, d["K"], k, oi, oc, bb, ov)
        return launch_topk(jobs)

    def _select_sets(self, step: int, items):
        """Top sets for [(head, k)] at one step, returned as sorted index arrays."""
        import torch

        if not items:
            return []
        kmax = max(1, max(k for _, k in items))
        out = torch.zeros((len(items), kmax), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(len(items), dtype=torch.int32, device="cuda")
        reqs = [(step, hd, k, _lib.ptr(out) + i * kmax * 4, _lib.ptr(cnt) + i * 4, 0, 0)
                for i, (hd, k) in enumerate(items)]
        jobs = self._select(reqs)
        o = out.cpu().numpy().view(np.uint32)
        c = cnt.cpu().numpy()
        del jobs
        return [np.sort(o[i, :c[i]]) for i in range(len(items))]

    def _upload_dynamic(self, hd, members) -> None:
        d = self._device()
        import torch

        bm = np.zeros(d["words"], dtype=np.uint32)
        arr = np.fromiter(members, dtype=np.int64, count=len(members))
        np.bitwise_or.at(bm, arr >> 5, (np.uint32(1) << (arr & 31).astype(np.uint32)))
        d["dyn_bm"][d["comp_slot"][hd]].copy_(torch.from_numpy(bm.view(np.int32)), non_blocking=False)

    # ---- primitives (engine.py:218-259) ------------------------------------

    def effective_length(self, head_id) -> int:
        if self.config.variant == "no_allocation":
            return self.l_base_int
        return self.plan.lengths[head_id]

    def _top_set(self, step: int, head_id, k: int) -> frozenset:
        return frozenset(int(x) for x in self._select_sets(step, [(head_id, k)])[0])

    def pivot_top_set(self, step: int, pivot) -> frozenset:
        top = self._top_set(step, pivot, self.l_base_int)
        if len(top) < self.l_base_int:
            raise InfeasibleStateError(
                f"pivot {pivot} recorded only {len(top)} live entries at step "
                f"{step}, monitoring needs {self.l_base_int}")
        return top

    def pivot_overlap(self, state: CacheState, pivot, step: int) -> float:
        return len(self.pivot_top_set(step, pivot) & state.k_base[pivot]) / self.l_base_int

    @staticmethod
    def drift_check(values, tau_drift: float) -> bool:
        """engine.py:247-250: window median strictly below tau (float64)."""
        return bool(np.median(list(values)) < tau_drift)

    def gpu_view(self, state: CacheState, head_id, step: int) -> CacheView:
        return CacheView(prefill_len=self.trace.manifest.prefill_len, step=step,
                         base=None if head_id in self.full else state.dynamic[head_id],
                         sink_count=self.config.sink_count,
                         recency_window=self.config.recency_window)

    # ---- lifecycle ----------------------------------------------------------

    def prefill_init(self) -> CacheState:
        state = CacheState(step=0, dynamic={}, k_base={}, buffers={}, buffer_steps={})
        d = self._device()
        monitor = self.config.variant != "no_retrieval"
        items = [(hd, self.effective_length(hd)) for hd in self.comp]
        if monitor:
            items += [(p, self.l_base_int) for p in self.pivots]
        sets = self._select_sets(0, items)
        for (hd, _), s in zip(items[:len(self.comp)], sets):
            state.dynamic[hd] = frozenset(int(x) for x in s)
            self._upload_dynamic(hd, state.dynamic[hd])
        if monitor:
            import torch

            for (p, _), s in zip(items[len(self.comp):], sets[len(self.comp):]):
                if len(s) < self.l_base_int:
                    raise InfeasibleStateError(
                        f"pivot {p} recorded only {len(s)} live entries at step 0, "
                        f"monitoring needs {self.l_base_int}")
                state.k_base[p] = frozenset(int(x) for x in s)
                bm = np.zeros(d["words"], dtype=np.uint32)
                np.bitwise_or.at(bm, s.astype(np.int64) >> 5,
                                 np.uint32(1) << (s & 31).astype(np.uint32))
                d["kbase_bm"][d["piv_slot"][p]].copy_(torch.from_numpy(bm.view(np.int32)))
                state.buffers[p] = []
                state.buffer_steps[p] = []
        return state

    def _measure_launch(self, step: int):
        d = self._device()
        m = self.trace.manifest
        _lib.check(_lib.load().hc_trace_recall(
            _lib.ptr(d["recall_heads"]), len(self.heads), d["K"], d["stride"], m.prefill_len,
            step, self.config.sink_count, self.config.recency_window, _lib.ptr(d["recall"]),
            _lib.stream_handle()))

    def _measure_finish(self, state: CacheState, step: int, recalls: np.ndarray) -> tuple:
        m = self.trace.manifest
        total = 0
        for hd in self.heads:
            total += self.gpu_view(state, hd, step).size()
        charged = len(self.full) * m.prefill_len + sum(len(state.dynamic[h]) for h in self.comp)
        recall = sum(recalls.tolist()) / len(self.heads)
        return recall, charged, total - charged

    def _measure(self, state: CacheState, step: int) -> tuple:
        self._measure_launch(step)
        return self._measure_finish(state, step, self._device()["recall"].cpu().numpy())

    def decode_step(self, state: CacheState, step: int) -> StepRow:
        cfg = self.config
        d = self._device()
        due = sorted((tr for tr in state.pending if tr.completion_step <= step),
                     key=lambda tr: (tr.completion_step, tr.order))
        state.pending = [tr for tr in state.pending if tr.completion_step > step]
        for tr in due:
            state.dynamic[tr.satellite] = tr.indices
        for s in {tr.satellite for tr in due}:
            self._upload_dynamic(s, state.dynamic[s])
        state.step = step

        # one launch for recall, one for every pivot's top set + overlap
        self._measure_launch(step)
        monitor = cfg.variant != "no_retrieval" and self.pivots
        jobs = None
        if monitor:
            reqs = []
            kc = d["kcap"]
            for p in self.pivots:
                i = d["piv_slot"][p]
                reqs.append((step, p, self.l_base_int, _lib.ptr(d["top_idx"]) + i * kc * 4,
                             _lib.ptr(d["top_cnt"]) + i * 4,
                             _lib.ptr(d["kbase_bm"]) + i * d["words"] * 4,
                             _lib.ptr(d["ovl"]) + i * 4))
            jobs = self._select(reqs)
        recalls = d["recall"].cpu().numpy()  # the step's one host sync
        recall, charged, extra = self._measure_finish(state, step, recalls)
        flag = 0
        if monitor:
            counts = d["top_cnt"].cpu().numpy()
            overlaps = d["ovl"].cpu().numpy()
            del jobs
            for p in self.pivots:
                i = d["piv_slot"][p]
                if counts[i] < self.l_base_int:
                    raise InfeasibleStateError(
                        f"pivot {p} recorded only {counts[i]} live entries at step "
                        f"{step}, monitoring needs {self.l_base_int}")
                state.buffers[p].append(int(overlaps[i]) / self.l_base_int)
                state.buffer_steps[p].append(step)
            for p in self.pivots:
                ready = (len(state.buffers[p]) >= cfg.window) if cfg.eval_every_step \
                    else (step % cfg.window == 0)
                if not ready:
                    continue
                fired = self.drift_check(state.buffers[p][-cfg.window:], cfg.tau_drift)
                if fired:
                    flag = 1
                    self._fire(state, p, step)
                if fired or not cfg.eval_every_step:
                    state.buffers[p] = []
                    state.buffer_steps[p] = []
        return StepRow(step=step, recall=recall, gpu_entries=charged, extra_entries=extra,
                       bytes_in_flight=state.bytes_in_flight(step),
                       cumulative_bytes=state.cumulative_bytes, retrieval_flag=flag)

    def _fire(self, state: CacheState, p, step: int) -> None:
        """engine.py:322-357: fetch selection on the GPU, accounting on the host."""
        cfg = self.config
        d = self._device()
        sats = self.satellites_of[p]
        sel = self._select_sets(step, [(p, self.effective_length(s)) for s in sats])
        fetches = [(s, tuple(int(x) for x in ix)) for s, ix in zip(sats, sel)]
        nbytes = sum(len(ix) for _, ix in fetches) * self.trace.manifest.bytes_per_kv_entry
        state.cumulative_bytes += nbytes
        done = completion_step(step, state.cumulative_bytes, cfg)
        for s, ix in fetches:
            state.pending.append(_Transfer(done, state._order_counter, s, frozenset(ix)))
            state._order_counter += 1
        state.events.append(RetrievalRecord(trigger_step=step, pivot=p, completion_step=done,
                                            transfer_bytes=nbytes, fetches=tuple(fetches)))
        # K_base <- current top set, on the device (engine.py:357)
        i = d["piv_slot"][p]
        _lib.check(_lib.load().hc_bitmap_from_indices(
            _lib.ptr(d["kbase_bm"]) + i * d["words"] * 4, d["words"],
            _lib.ptr(d["top_idx"]) + i * d["kcap"] * 4, _lib.ptr(d["top_cnt"]) + i * 4,
            d["kcap"], _lib.stream_handle()))
        cnt = int(d["top_cnt"][i].item())
        cur = d["top_idx"][i, :cnt].cpu().numpy().view(np.uint32)
        state.k_base[p] = frozenset(int(x) for x in cur)

    def run(self) -> EngineRun:
        m = self.trace.manifest
        state = self.prefill_init()
        recall, charged, extra = self._measure(state, 0)
        rows = [StepRow(step=0, recall=recall, gpu_entries=charged, extra_entries=extra,
                        bytes_in_flight=0, cumulative_bytes=0, retrieval_flag=0)]
        for step in range(1, m.decode_steps + 1):
            rows.append(self.decode_step(state, step))
        final_gpu = {}
        L, T = m.prefill_len, m.decode_steps
        for hd in self.heads:
            members = set(range(L, L + T))
            members.update(range(min(self.config.sink_count, L)))
            members.update(range(max(0, L + T - self.config.recency_window), L))
            members.update(range(L) if hd in self.full else state.dynamic[hd])
            final_gpu[hd] = frozenset(members)
        report = SimulationReport(
            policy=self.config.variant, trace_sha256=trace_fingerprint(self.trace),
            num_layers=m.num_layers, heads_per_layer=m.heads_per_layer, prefill_len=L,
            decode_steps=T, budget_ceiling=self.plan.budget_ceiling,
            update_delay_steps=self.config.update_delay_steps, rows=tuple(rows),
            events=tuple(state.events))
        return EngineRun(report=report, final_gpu=final_gpu, state=state)


def run_simulation(trace, taxonomy, plan, config: EngineConfig = EngineConfig()) -> EngineRun:
    return CacheEngine(trace, taxonomy, plan, config).run()
