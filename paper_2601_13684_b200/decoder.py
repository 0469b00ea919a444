"""Tensor-mode HeteroCache decoder: the reference engine's logic over real K/V.

``HeteroCacheDecoder`` owns one engine handle (libhcb200.so) holding the
hierarchical KV store for a batch of sequences.  Each sequence behaves as one
reference ``CacheEngine`` (engine.py:153-416) sharing the taxonomy and plan:

  prefill_layer(l, K, V, q_last)      prefill_init  (engine.py:263-274)
  decode_step(t, q, k_new, v_new, o)  decode_step   (engine.py:290-370)

Per decode step the GPU appends the new token, runs the fused ragged
flash-decoding kernel over every resident set, forms the pivots' GQA-mean
probability rows and their top-l_base sets with |top & K_base| counts.  The
host keeps exactly the reference's bookkeeping per sequence: the window
buffers and median test (engine.py:305-321), byte accounting and completion
steps (engine.py:322-347), FIFO landing of due transfers (engine.py:293-299)
and the StepRow / RetrievalRecord records (reporting.py).  Host <-> device
synchronisation happens only at window boundaries (or every step with
eval_every_step), where the overlap counts are read back -- and, with
overlap_decisions (default), not even there on the GPU's critical path: the
boundary decision of step t is taken inside step t+1, while that step's
attention over every non-satellite head already runs (decode_begin /
decode_end), so its StepRow and events appear one step later or at finish().

StepRow.recall is NaN unless measure mode is on (recall_topk > 0):
attention-mass recall (evaluation.py:41-59) needs every head's full attention,
which the compressed path by design never computes.  In measure mode the
engine keeps a full-context K copy, forms every head's dense row per step,
records its top recall_topk positions (step 0 and pivots: enough records for
every selection the reference makes from them; pivots use their own decision
rows) and computes each head's recall of the recorded
mass against its resident set on the GPU -- the records are exactly an
HCTRACE1 trace of the run (tools/export_trace.py), so the reference engine
replaying it reproduces the StepRows bit for bit.
"""

from __future__ import annotations

import ctypes as C
import math
from collections import deque
from dataclasses import dataclass, field
from math import ceil

import numpy as np

from . import _lib
from .engine import EngineConfig, EngineError, InfeasibleStateError, completion_step
from .reporting import RetrievalRecord, SimulationReport, StepRow

ROLE_CODE = {"volatile": 0, "anchor": 1, "pivot": 2, "satellite": 3}


def window_median(v: np.ndarray) -> np.ndarray:
    """Column medians of a [W, m] float64 window, bit-identical to np.median(axis=0)
    (middle element, or (a + b) / 2 of the middle pair: numpy's mean of two)."""
    s = np.sort(v, axis=0)
    n = s.shape[0]
    if n % 2:
        return s[n // 2]
    return (s[n // 2 - 1] + s[n // 2]) / 2


@dataclass
class _Event:
    """A fired retrieval; fetched sets arrive asynchronously (pinned D2H)."""

    trigger_step: int
    pivot: tuple
    completion_step: int
    transfer_bytes: int
    sats: tuple
    ks: list
    tids: list = field(default_factory=list)
    offsets: list = field(default_factory=list)
    fetched: list = None

    def record(self) -> RetrievalRecord:
        if self.fetched is None:
            raise EngineError("fetched sets not yet available: call decoder.sync() first")
        return RetrievalRecord(
            trigger_step=self.trigger_step, pivot=self.pivot,
            completion_step=self.completion_step, transfer_bytes=self.transfer_bytes,
            fetches=tuple((s, tuple(int(x) for x in f)) for s, f in zip(self.sats, self.fetched)))


@dataclass
class SequenceState:
    """Per-sequence mirror of CacheState (engine.py:126-143)."""

    step: int = 0
    buffers: dict = field(default_factory=dict)       # pivot -> overlap values (sliding mode)
    pending: list = field(default_factory=list)       # (completion, order, sat, tid, k, event)
    raw_events: list = field(default_factory=list)    # _Event, trigger order
    cumulative_bytes: int = 0
    ledger: list = field(default_factory=list)        # (completion, bytes) of every event, all ranks
    order: int = 0
    dyn_count: dict = field(default_factory=dict)     # compressed head -> |dynamic|
    dyn_sets: dict = field(default_factory=dict)      # compressed head -> sorted positions
    rows: list = field(default_factory=list)

    @property
    def events(self) -> list:
        """RetrievalRecords (reporting.py:58-91), materialised on demand."""
        return [e.record() for e in self.raw_events]

    def bytes_in_flight(self, step: int) -> int:
        return sum(n for c, n in self.ledger if c > step)


class HeteroCacheDecoder:
    def __init__(self, taxonomy, plan, config: EngineConfig = EngineConfig(), *, batch: int,
                 group: int, max_decode: int, head_dim: int = 128, chunk: int = 1024,
                 host_pool: bool = True, bytes_per_kv_entry: int | None = None,
                 track_sets: bool = True, obs_window: int = 1, overlap_decisions: bool = True,
                 recall_topk: int = 0, owned=None, exchange=None,
                 score_material: str = "fp32", fetch_ring_entries: int | None = None,
                 device_decisions: bool | None = None):
        """owned: optional [batch, layers, kv_heads] bool mask of the units this
        rank holds (parallel.assign_units; None = all).  exchange: the fire
        exchange of a unit-sharded run (parallel.FireExchange); every rank of
        the run must step in lockstep, since boundary decisions all_gather.
        score_material: "fp32" (default) or "fp16", the per-token pivot material
        K4 hands to the GQA-mean row pass; fp16 halves those bytes but its
        ~5e-4 relative row error moves near-tied positions across the top-k
        boundary (profiles/r02_selection_precision.json).
        fetch_ring_entries: size of the pinned ring the fetched sets land in
        (default: four full drift bursts, at least 64K entries).
        device_decisions: take the boundary decisions on the device (devdec.cu:
        window median, accounting, fetch selection, gathers, landings in device
        streams; this mirror reads them from a mapped log without ever blocking
        the step).  None (default) = on whenever supported: monitored pivots, an
        unsharded engine, no measure mode, window <= 64."""
        _lib.require_cuda()
        self.lib = _lib.load()
        self.taxonomy, self.plan, self.config = taxonomy, plan, config
        self.B, self.NL, self.H = batch, taxonomy.num_layers, taxonomy.heads_per_layer
        self.G, self.D, self.L, self.T = group, head_dim, plan.prefill_len, max_decode
        self.bytes_per_entry = bytes_per_kv_entry or 2 * head_dim * 2  # export.ts:104
        self.track_sets = track_sets
        self.full = set(taxonomy.full_heads())
        self.comp = list(taxonomy.compressed_heads())
        if set(plan.lengths) != set(self.comp):
            raise EngineError("plan does not cover exactly the compressed heads")
        self.pivots = list(taxonomy.pivots())
        self.satellites_of = {p: tuple(taxonomy.cluster_of(p).satellites) for p in self.pivots}
        self.l_base_int = plan.l_base_int
        if self.l_base_int < 1:
            raise InfeasibleStateError(f"per-head base budget rounds to {self.l_base_int}")
        self.monitor = bool(self.pivots) and config.variant != "no_retrieval"
        LH = self.NL * self.H
        roles = np.zeros(LH, dtype=np.int32)
        lengths = np.zeros(LH, dtype=np.int32)
        cpiv = np.full(LH, -1, dtype=np.int32)
        for (l, h), prof in taxonomy.heads.items():
            roles[l * self.H + h] = ROLE_CODE[prof.role]
            if (l, h) in plan.lengths:
                lengths[l * self.H + h] = self.effective_length((l, h))
        for p, sats in self.satellites_of.items():
            for s in sats:
                cpiv[s[0] * self.H + s[1]] = p[1]
        most_sats = max((len(s) for s in self.satellites_of.values()), default=0)
        ok_dev = (self.monitor and owned is None and not recall_topk and config.window <= 64
                  and len(plan.lengths) > 0 and most_sats <= 8)
        if device_decisions and not ok_dev:
            raise EngineError("device decisions need monitored pivots, an unsharded engine, "
                              "no measure mode, window <= 64 and at most 8 satellites per pivot")
        self.devdec = ok_dev if device_decisions is None else bool(device_decisions)
        desc = _lib.EngineDesc(batch=batch, num_layers=self.NL, kv_heads=self.H, group=group,
                               head_dim=head_dim, prefill_len=self.L, max_decode=max_decode,
                               sink_count=config.sink_count, recency_window=config.recency_window,
                               l_base_int=self.l_base_int, chunk=chunk, monitor=int(self.monitor),
                               host_pool=int(host_pool), obs_window=obs_window,
                               score_material={"fp32": 0, "fp16": 1}[score_material],
                               device_decisions=int(self.devdec), window=config.window,
                               update_delay_steps=config.update_delay_steps,
                               eval_every_step=int(config.eval_every_step),
                               bytes_per_kv_entry=self.bytes_per_entry,
                               transfer_bandwidth=int(config.transfer_bandwidth),
                               tau_drift=float(config.tau_drift))
        self.W = obs_window
        h = C.c_void_p()
        if owned is None:
            self.owned = np.ones((batch, self.NL, self.H), dtype=bool)
            _lib.check(self.lib.hc_engine_create(C.byref(desc), roles.ctypes.data,
                                                 lengths.ctypes.data, cpiv.ctypes.data, C.byref(h)))
        else:
            self.owned = np.ascontiguousarray(np.asarray(owned, dtype=bool).reshape(
                batch, self.NL, self.H))
            om = self.owned.astype(np.uint8)
            _lib.check(self.lib.hc_engine_create_sharded(C.byref(desc), roles.ctypes.data,
                                                         lengths.ctypes.data, cpiv.ctypes.data,
                                                         om.ctypes.data, C.byref(h)))
        self.handle = h
        if exchange is None:
            from .parallel import LocalExchange

            exchange = LocalExchange()
        self.exchange = exchange
        # per sequence: the heads / pivots this rank holds (all of them unsharded)
        own = self.owned
        self.full_of = [[hd for hd in sorted(self.full) if own[b][hd]] for b in range(batch)]
        self.comp_of = [[hd for hd in self.comp if own[b][hd]] for b in range(batch)]
        self.piv_of = [[p for p in self.pivots if own[b][p]] for b in range(batch)]
        # measure mode (recall at scale): every head's top-recall_topk records per step
        self.recall_topk = recall_topk
        self.record_k = max([recall_topk, self.l_base_int if self.monitor else 0] +
                            [self.effective_length(hd) for hd in self.comp])
        if recall_topk:
            _lib.check(self.lib.hc_engine_enable_measure(self.handle, recall_topk))
        info = (C.c_int64 * 4)()
        _lib.check(self.lib.hc_engine_info(self.handle, info))
        self.device_bytes, self.host_bytes, self.arena_rows, self.n_pivot_units = list(info)
        # pivot slot order == ascending unit order
        self.pivot_units = [self.unit(b, p) for b in range(self.B) for p in self.piv_of[b]] \
            if self.monitor else []
        self.pivot_units.sort()
        self.pivot_slot = {u: i for i, u in enumerate(self.pivot_units)}
        self.states = [SequenceState() for _ in range(self.B)]
        if self.devdec:  # the device mirror pops landings / landed ledger entries in order
            for st in self.states:
                st.pending, st.ledger = deque(), deque()
        self._cols = [[self.pivot_slot[self.unit(b, p)] for p in self.piv_of[b]] if self.monitor
                      else [] for b in range(self.B)]
        self._pinned = None
        self._pin_head = 0
        self._ring_entries = fetch_ring_entries
        self._fetch_pending = False
        self._uncollected = []
        np.median(np.zeros((2, 2)), axis=0)  # first call imports numpy.ma (~30 ms): not mid-run
        self._prefilled = set()
        # boundary decision taken while the next step's attention runs (see
        # decode_step); (step, first, per-sequence (charged, extra)) or None
        self.overlap_decisions = overlap_decisions
        self._open = None
        # device decisions: steps not yet turned into StepRows, boundaries not yet read
        self._dd_steps = deque()  # (t, boundary, rows)
        self._dd_unread = []      # boundary steps issued, decision not read yet
        self._dd_fired = {}       # boundary step -> sequences that fired
        if self.devdec:
            n = C.c_int32()
            _lib.check(self.lib.hc_engine_devdec_satellites(self.handle, None, 0, C.byref(n)))
            su = np.zeros(max(1, n.value), dtype=np.int32)
            _lib.check(self.lib.hc_engine_devdec_satellites(self.handle, su.ctypes.data,
                                                            su.size, C.byref(n)))
            LHn = self.NL * self.H
            self._dd_sat_head = [((int(u) % LHn) // self.H, int(u) % self.H)
                                 for u in su[:n.value]]
            self._dd_recs = (_lib.FireRecord * max(1, self.n_pivot_units))()
            cap = sum(self.effective_length(s) for b in range(self.B) for p in self.piv_of[b]
                      for s in self.satellites_of[p])
            self._dd_fetched = np.empty(max(1, cap), dtype=np.uint32)
            # per-step call path: bound C entry points and reusable out-arguments
            self._c_step, self._c_nf = C.c_int32(), C.c_int32()
            self._poll_args = (C.byref(self._c_step), self._dd_recs, len(self._dd_recs),
                               C.byref(self._c_nf), self._dd_fetched.ctypes.data,
                               self._dd_fetched.size)
        self._pinned_ok = set()  # (data_ptr, nbytes) of host tensors decode_step_host checked

    # ---- helpers -------------------------------------------------------------

    def unit(self, b: int, head_id) -> int:
        l, h = head_id
        return (b * self.NL + l) * self.H + h

    def effective_length(self, head_id) -> int:
        if self.config.variant == "no_allocation":
            return self.l_base_int
        return self.plan.lengths[head_id]

    def close(self):
        if getattr(self, "handle", None):
            self.lib.hc_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def read_indices(self, kind: int, ident: int, capacity: int, stream=None) -> np.ndarray:
        out = np.empty(max(1, capacity), dtype=np.uint32)
        n = C.c_int32()
        _lib.check(self.lib.hc_engine_read_indices(self.handle, kind, ident, out.ctypes.data,
                                                   capacity, C.byref(n), _lib.stream_handle(stream)))
        return np.sort(out[:n.value])

    def dynamic_set(self, b: int, head_id) -> np.ndarray:
        return self.read_indices(1, self.unit(b, head_id), self.L + self.T)

    def prefix_positions(self, b: int, head_id) -> np.ndarray:
        """Positions held in a compressed unit's active prefix buffer (storage order)."""
        out = np.empty(self.L + self.T, dtype=np.uint32)
        n = C.c_int32()
        _lib.check(self.lib.hc_engine_read_indices(self.handle, 3, self.unit(b, head_id),
                                                   out.ctypes.data, out.size, C.byref(n),
                                                   _lib.stream_handle()))
        return out[:n.value].copy()

    def pivot_top_set(self, b: int, pivot) -> np.ndarray:
        return self.read_indices(2, self.unit(b, pivot), self.l_base_int)

    # ---- prefill (engine.py:263-274) --------------------------------------------

    def prefill_layer(self, layer: int, k, v, q_last, stream=None) -> None:
        """k, v: [B, H, L, D] bf16 device tensors; q_last: [B, H*G, D] bf16 (window 1)
        or [B, w, H*G, D] (observation window w)."""
        qshape = (self.B, self.H * self.G, self.D) if self.W == 1 else \
            (self.B, self.W, self.H * self.G, self.D)
        for t, shape in ((k, (self.B, self.H, self.L, self.D)), (v, (self.B, self.H, self.L, self.D)),
                         (q_last, qshape)):
            if tuple(t.shape) != shape or not t.is_contiguous() or not t.is_cuda:
                raise EngineError(f"expected a contiguous CUDA tensor of shape {shape}")
        _lib.check(self.lib.hc_engine_prefill_layer(self.handle, layer, _lib.ptr(k), _lib.ptr(v),
                                                    _lib.ptr(q_last), _lib.stream_handle(stream)))
        self._prefilled.add(layer)

    def finish_prefill(self) -> None:
        """Build the host mirror once every layer is prefilled (reads the sets back)."""
        if len(self._prefilled) != self.NL:
            raise EngineError("prefill every layer before decoding")
        for b, st in enumerate(self.states):
            for hd in self.comp_of[b]:
                k = self.effective_length(hd)
                st.dyn_count[hd] = min(k, self.L)
                if self.track_sets:
                    st.dyn_sets[hd] = self.dynamic_set(b, hd)
            if self.monitor:
                for p in self.piv_of[b]:
                    st.buffers[p] = []
        rec = self._measure(0, None)
        for b, st in enumerate(self.states):
            st.rows.append(self._row(st, 0, 0, self._row_sizes(b, 0, rec[b])))
        if self.monitor:  # pinned landing zone for fetched sets: every satellite firing at once
            import torch

            cap = sum(self.effective_length(s) for b in range(self.B) for p in self.piv_of[b]
                      for s in self.satellites_of[p])
            n = self._ring_entries or max(4 * cap, 1 << 16)  # four full drift bursts
            self._pinned = torch.empty(max(n, cap), dtype=torch.int32, pin_memory=True)
            self._pin_head = 0

    # ---- decode -------------------------------------------------------------------

    def _size_of(self, st: SequenceState, hd, t: int) -> int:
        """CacheView.size (engine.py:109-115) from the host mirror."""
        L, S, R = self.L, self.config.sink_count, self.config.recency_window
        extras = set(range(min(S, L))) | set(range(max(0, L + t - R), L))
        dyn = st.dyn_sets.get(hd)
        if dyn is None:
            return -1
        inter = int(np.isin(np.fromiter(extras, dtype=np.int64, count=len(extras)), dyn).sum())
        return len(dyn) + len(extras) - inter + t

    def _row_sizes(self, b: int, t: int, recall: float = math.nan):
        """(charged, extra, recall) of sequence b at step t over the heads this
        rank holds (engine.py:276-288); a unit-sharded run adds the ranks'
        partials (parallel.merge_reports)."""
        st = self.states[b]
        nf = len(self.full_of[b])
        charged = nf * self.L + sum(st.dyn_count.values())
        if self.track_sets:
            total = nf * (self.L + t) + sum(self._size_of(st, hd, t) for hd in self.comp_of[b])
            extra = total - charged
        else:
            extra = -1
        return charged, extra, recall

    def _measure(self, t: int, q, sh=None) -> list:
        """Per-sequence recall at step t (CacheEngine._measure, engine.py:276-288):
        the mean over heads in (layer, head) order of each head's recall of its
        recorded mass; NaN when measure mode is off."""
        if not self.recall_topk:
            return [math.nan] * self.B
        out = np.empty(self.B * self.NL * self.H, dtype=np.float64)
        _lib.check(self.lib.hc_engine_measure(self.handle, t, _lib.ptr(q) if q is not None else None,
                                              out.ctypes.data,
                                              sh if sh is not None else _lib.stream_handle()))
        per = out.reshape(self.B, self.NL * self.H)
        return [sum(per[b].tolist()) / (self.NL * self.H) for b in range(self.B)]

    def measure_records(self, b: int, head_id):
        """(indices, scores) recorded for one head at the last measured step."""
        cap = self.record_k
        idx = np.empty(cap, dtype=np.uint32)
        sc = np.empty(cap, dtype=np.float32)
        _lib.check(self.lib.hc_engine_measure_records(self.handle, self.unit(b, head_id),
                                                      idx.ctypes.data, sc.ctypes.data, cap,
                                                      _lib.stream_handle()))
        return idx, sc

    def _row(self, st: SequenceState, t: int, flag: int, sizes) -> StepRow:
        charged, extra, recall = sizes
        return StepRow(step=t, recall=recall, gpu_entries=charged, extra_entries=extra,
                       bytes_in_flight=st.bytes_in_flight(t), cumulative_bytes=st.cumulative_bytes,
                       retrieval_flag=flag)

    def _land_due(self, t: int, sh) -> None:
        """Land due transfers (engine.py:293-299): per sequence in (completion,
        order) order, all sequences in one batched call."""
        land = []
        for st in self.states:
            if st.pending and st.pending[0][0] <= t:  # pending is kept sorted
                k = 0
                while k < len(st.pending) and st.pending[k][0] <= t:
                    _, _, s, tid, n, ev = st.pending[k]
                    land.append(tid)
                    st.dyn_count[s] = n
                    if self.track_sets:
                        st.dyn_sets[s] = ev.fetched[ev.tids.index(tid)]
                    k += 1
                del st.pending[:k]
            st.step = t
        if land:
            ids = np.asarray(land, dtype=np.int32)
            _lib.check(self.lib.hc_engine_land_batch(self.handle, len(ids), ids.ctypes.data, sh))

    def decode_step(self, t: int, q, k_new, v_new, out, stream=None, *, rows: bool = True):
        """q/out: [B, NL, H*G, D] bf16; k_new/v_new: [B, NL, H, D] bf16 (device).

        With overlap_decisions (default) a window boundary's decision (median
        test, firing, engine.py:313-360) is taken inside the NEXT step, after
        that step's attention over every non-satellite head is queued: the
        host work and the fetch selection then overlap the GPU instead of
        idling it.  Semantics are unchanged -- the decision reads step t's
        counts and rows, its transfers land at their completion steps -- but
        the StepRow / events of boundary step t appear when step t+1 runs (or
        at finish()).
        """
        cfg = self.config
        sh = _lib.stream_handle(stream)
        if self.devdec:
            rc = self.lib.hc_engine_decode_step(self.handle, t, q.data_ptr(), k_new.data_ptr(),
                                                v_new.data_ptr(), out.data_ptr(), sh)
            if rc:
                _lib.check(rc)
            self._dd_after_step(t, rows)
            return
        hold = self._open is not None
        self._land_due(t, sh)
        if hold:
            _lib.check(self.lib.hc_engine_decode_begin(self.handle, t, _lib.ptr(q),
                                                       _lib.ptr(k_new), _lib.ptr(v_new),
                                                       _lib.ptr(out), 1, sh))
            self._close_decision(sh)
            self._land_due(t, sh)  # transfers the decision completes at t
            _lib.check(self.lib.hc_engine_decode_end(self.handle, t, sh))
        else:
            _lib.check(self.lib.hc_engine_decode_step(self.handle, t, _lib.ptr(q), _lib.ptr(k_new),
                                                      _lib.ptr(v_new), _lib.ptr(out), sh))
        rec = self._measure(t, q, sh) if self.recall_topk else [math.nan] * self.B
        boundary = self.monitor and (cfg.eval_every_step or t % cfg.window == 0)
        if boundary:
            first = t if cfg.eval_every_step else max(1, t - cfg.window + 1)
            self._open = (t, first, [self._row_sizes(b, t, rec[b])
                                     for b in range(self.B)] if rows else None)
            if not self.overlap_decisions:
                self._close_decision(sh)
        elif rows:
            for b, st in enumerate(self.states):
                st.rows.append(self._row(st, t, 0, self._row_sizes(b, t, rec[b])))

    def decode_step_host(self, t: int, q, k_new, v_new, out, stream=None, *, rows: bool = True):
        """decode_step from pinned host tensors (a serving runtime's per-step call,
        hc_engine_decode_step_host): the inputs cross H2D and the output D2H on
        the engine's copy stream; `out` holds step t once `stream` has passed
        join().  Needs device decisions."""
        if not self.devdec:
            raise EngineError("decode_step_host needs device decisions")
        for x in (q, k_new, v_new, out):
            if x.is_cuda or not x.is_contiguous():
                raise EngineError("decode_step_host takes contiguous pinned host tensors")
            key = (x.data_ptr(), x.nbytes)
            if key in self._pinned_ok:  # (is_pinned() queries the driver: once per buffer)
                continue
            if not x.is_pinned():
                raise EngineError("decode_step_host takes contiguous pinned host tensors")
            if len(self._pinned_ok) > 256:
                self._pinned_ok.clear()
            self._pinned_ok.add(key)
        rc = self.lib.hc_engine_decode_step_host(
            self.handle, t, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
            _lib.stream_handle(stream))
        if rc:
            _lib.check(rc)
        self._dd_after_step(t, rows)

    # ---- device decisions: the host mirror ----------------------------------------

    def _dd_after_step(self, t: int, rows: bool) -> None:
        cfg = self.config
        boundary = cfg.eval_every_step or t % cfg.window == 0
        self._dd_steps.append((t, boundary, rows))
        if boundary:
            self._dd_unread.append(t)
        # read whatever the device has decided by now; block (on a decision
        # several boundaries old -- the GPU still has those steps queued) only
        # when more than 4 are unread: the mapped fetched-set ring holds 6
        # boundaries of every satellite firing
        self._dd_poll(keep=4)

    def _dd_poll(self, keep: int = 0) -> None:
        """Read device decisions in boundary order -- those already done, and
        blocking on the oldest while more than `keep` are unread -- and turn the
        steps they complete into StepRows."""
        step, nf = self._c_step, self._c_nf
        while self._dd_unread:
            wait = len(self._dd_unread) > keep
            _lib.check(self.lib.hc_engine_poll_decisions(self.handle, int(wait),
                                                         *self._poll_args))
            if step.value < 0:
                break
            t = step.value
            if t != self._dd_unread[0]:
                raise EngineError(f"device decision for step {t}, expected {self._dd_unread[0]}")
            self._dd_materialise(upto=t - 1)  # rows before t must not see t's fires
            self._dd_unread.pop(0)
            self._dd_record(t, nf.value)
        self._dd_materialise()

    def _dd_record(self, t: int, n: int) -> None:
        """RetrievalRecords and pending landings of boundary t's fires (device order:
        per sequence, sorted pivots -- engine.py:313)."""
        LHn = self.NL * self.H
        fired = set()
        for i in range(n):
            r = self._dd_recs[i]
            b = r.pivot_unit // LHn
            p = ((r.pivot_unit % LHn) // self.H, r.pivot_unit % self.H)
            sats = tuple(self._dd_sat_head[r.first_satellite + j] for j in range(r.n_satellites))
            ks = [int(r.fetched_counts[j]) for j in range(r.n_satellites)]
            if r.fetched_offset < 0:
                raise EngineError("device decisions: fetched sets unavailable")
            fetched, o = [], r.fetched_offset
            for k in ks:
                fetched.append(self._dd_fetched[o:o + k].copy())
                o += k
            st = self.states[b]
            ev = _Event(trigger_step=t, pivot=p, completion_step=r.completion_step,
                        transfer_bytes=int(r.transfer_bytes), sats=sats, ks=ks, fetched=fetched)
            st.raw_events.append(ev)
            # completion steps never decrease in firing order (cumulative bytes
            # only grow): the pending deque stays in (completion, order) order
            for s, k, f in zip(sats, ks, fetched):
                st.pending.append((r.completion_step, st.order, s, -1, k, ev))
                st.order += 1
            st.cumulative_bytes = int(r.cumulative_bytes)
            while st.ledger and st.ledger[0][0] <= t - 1:  # landed: never in flight again
                st.ledger.popleft()
            st.ledger.append((r.completion_step, int(r.transfer_bytes)))
            fired.add(b)
        self._dd_fired[t] = fired

    def _dd_materialise(self, upto: int | None = None) -> None:
        """StepRows of every step whose decisions (and all earlier ones) are read
        (and, with upto, of steps <= upto only)."""
        first_unread = self._dd_unread[0] if self._dd_unread else None
        while self._dd_steps and (first_unread is None or self._dd_steps[0][0] < first_unread) \
                and (upto is None or self._dd_steps[0][0] <= upto):
            t, boundary, rows = self._dd_steps.popleft()
            for st in self.states:  # landings due at t (engine.py:293-299), before t's
                # own decision: a transfer fired at t lands at t + 1 at the earliest
                while st.pending and st.pending[0][0] <= t and st.pending[0][5].trigger_step < t:
                    _, _, s, _, n_, ev = st.pending.popleft()
                    st.dyn_count[s] = n_
                    if self.track_sets:
                        st.dyn_sets[s] = ev.fetched[ev.sats.index(s)]
                st.step = t
            fired = self._dd_fired.pop(t, set()) if boundary else set()
            if rows:
                for b, st in enumerate(self.states):
                    st.rows.append(self._row(st, t, int(b in fired), self._row_sizes(b, t)))

    def _close_decision(self, sh) -> None:
        t, first, sizes = self._open
        self._open = None
        flags = [0] * self.B
        self._decide(t, first, flags, sh)
        if sizes is not None:
            for b, st in enumerate(self.states):
                st.rows.append(self._row(st, t, flags[b], sizes[b]))

    def finish(self, stream=None) -> None:
        """Take a still-open boundary decision (the last decoded step's); with
        device decisions, read all of them."""
        if self.devdec:
            self._dd_poll(keep=0)
            return
        if self._open is not None:
            self._close_decision(_lib.stream_handle(stream))

    def _decide(self, t: int, first: int, flags: list, sh) -> None:
        """Window median test and firing (engine.py:305-360), vectorised over pivots.

        Boundary mode: the buffers hold exactly this window's values (they are
        cleared at every boundary), so medians are one np.median over axis 0
        (same partition + mean-of-middle-pair arithmetic as the reference's
        per-list np.median).  Sliding mode keeps per-pivot lists.  The fires of
        every rank (one rank unsharded) are then accounted in the reference's
        sorted pivot order per sequence (parallel.order_fires).
        """
        from .parallel import order_fires

        cfg = self.config
        n = t - first + 1
        counts = np.empty((n, len(self.pivot_units)), dtype=np.int32)
        _lib.check(self.lib.hc_engine_overlaps(self.handle, first, t, counts.ctypes.data, sh))
        vals = counts / self.l_base_int  # float64, == int / int in Python
        med = None if cfg.eval_every_step else window_median(vals) < cfg.tau_drift
        local = []  # (b, pivot, sats, ks, bytes) in (b, sorted pivot) order
        for b, st in enumerate(self.states):
            cols = self._cols[b]
            pivs = self.piv_of[b]
            if cfg.eval_every_step:
                fired_mask = []
                for j, p in enumerate(pivs):
                    buf = st.buffers[p]
                    buf.extend(vals[:, cols[j]].tolist())
                    fired = len(buf) >= cfg.window and \
                        bool(np.median(buf[-cfg.window:]) < cfg.tau_drift)
                    if fired:
                        st.buffers[p] = []
                    fired_mask.append(fired)
            else:
                fired_mask = med[cols].tolist()
            for j, p in enumerate(pivs):
                if fired_mask[j]:
                    sats = self.satellites_of[p]
                    ks = [min(self.effective_length(s), self.L + t) for s in sats]
                    local.append((b, p, sats, ks, sum(ks) * self.bytes_per_entry))
        gathered = self.exchange.all_gather([(b, p, nb) for b, p, _, _, nb in local])
        if not any(gathered):
            return
        cum = [st.cumulative_bytes for st in self.states]
        done_of = order_fires(t, gathered, cum, cfg)
        # the fire selection and gathers first (the GPU is waiting for them), the
        # host bookkeeping after
        if local:
            issued = self._fire_batch(t, local, [done_of[(b, p)][0] for b, p, _, _, _ in local], sh)
        for b, _ in done_of:
            flags[b] = 1
        for st in self.states:  # landed transfers never count as in flight again
            st.ledger = [(c, n_) for c, n_ in st.ledger if c > t - 1]
        for b, p, n_ in sorted((b, p, n_) for part in gathered for (b, p, n_) in part):
            self.states[b].ledger.append((done_of[(b, p)][0], n_))
        for b, st in enumerate(self.states):
            st.cumulative_bytes = cum[b]
        if local:
            self._record_fires(t, local, done_of, *issued)

    def _fire_batch(self, t: int, local, done, sh):
        """hc_engine_fire_batch for this boundary's local fires: selection, K_base
        restamp, fetched-set copies into the pinned ring, gathers.  Returns the
        transfer ids and the ring offset of the batch."""
        total = sum(sum(ks) for _, _, _, ks, _ in local)
        self._reserve_pinned(total)
        base = self._pin_head
        ids = np.zeros(sum(len(sats) for _, _, sats, _, _ in local), dtype=np.int32)
        u = np.asarray([self.unit(b, p) for b, p, _, _, _ in local], dtype=np.int32)
        d = np.asarray(done, dtype=np.int32)
        _lib.check(self.lib.hc_engine_fire_batch(self.handle, len(u), u.ctypes.data, t,
                                                 d.ctypes.data, ids.ctypes.data,
                                                 self._pinned.data_ptr() + 4 * base, sh))
        self._pin_head = base + total
        self._fetch_pending = True  # hc_engine_wait_fetched marks the ring readable
        return ids, base

    def _record_fires(self, t: int, local, done_of, ids, base) -> None:
        """RetrievalRecords (engine.py:338-347) and pending landings of the fires
        just issued, in firing order."""
        q = 0
        off = base
        unsorted = []
        for b, p, sats, ks, nbytes in local:
            st = self.states[b]
            ev = _Event(trigger_step=t, pivot=p, completion_step=done_of[(b, p)][0],
                        transfer_bytes=nbytes, sats=sats, ks=ks)
            st.raw_events.append(ev)
            ev.tids = ids[q:q + len(sats)].tolist()
            ev.offsets = []
            for k in ks:
                ev.offsets.append((off, k))
                off += k
            q += len(sats)
            for s, k, tid in zip(sats, ks, ev.tids):
                if st.pending and st.pending[-1][0] > ev.completion_step and \
                        all(x is not st for x in unsorted):
                    unsorted.append(st)
                st.pending.append((ev.completion_step, st.order, s, tid, k, ev))
                st.order += 1
            self._uncollected.append(ev)
        # completion steps are nondecreasing in firing order (cumulative bytes only
        # grow), so appends keep the (completion, order) landing order of
        # engine.py:293-296; re-sort only if that ever does not hold
        for st in unsorted:
            st.pending.sort(key=lambda x: (x[0], x[1]))
        if self.track_sets:  # the host mirror needs the sets: wait for their copies only
            self._drain_fetched()

    def _reserve_pinned(self, total: int) -> None:
        """Fetched sets land in a pinned ring; collect lazily, only before reuse."""
        import torch

        if self._pinned is None or self._pinned.numel() < total:
            self._drain_fetched()
            self._pinned = torch.empty(max(total, 1 << 16), dtype=torch.int32, pin_memory=True)
            self._pin_head = 0
        if self._pin_head + total > self._pinned.numel():
            self._drain_fetched()  # copy out what the ring still holds before overwriting it
            self._pin_head = 0

    def _drain_fetched(self) -> None:
        """Wait for the copies into the ring (the engine's side-stream event of the
        last fire batch), not for the caller's queue, then copy the ring out."""
        if self._fetch_pending:
            _lib.check(self.lib.hc_engine_wait_fetched(self.handle))
            self._fetch_pending = False
        self._collect_fetched()

    def _collect_fetched(self) -> None:
        """Copy fetched index sets out of the pinned staging buffer (after a sync)."""
        if not self._uncollected:
            return
        import torch

        spans = [(o, o + k) for ev in self._uncollected for o, k in ev.offsets]
        lo = min(a for a, _ in spans) if spans else 0
        end = max((b for _, b in spans), default=0)
        # one bulk copy of just the uncollected span of the ring (torch's copy is
        # multithreaded: the ring can hold tens of MB)
        buf = torch.empty(end - lo, dtype=torch.int32)
        buf.copy_(self._pinned[lo:end])
        store = buf.numpy().view(np.uint32)
        for ev in self._uncollected:  # K1 dense output is already ascending
            ev.fetched = [store[o - lo:o - lo + k] for o, k in ev.offsets]
        self._uncollected = []

    def join(self, stream=None) -> None:
        """Order `stream` after the engine's side-stream work (the last monitor)."""
        _lib.check(self.lib.hc_engine_join(self.handle, _lib.stream_handle(stream)))

    def sync(self, stream=None) -> None:
        import torch

        self.finish(stream)
        self.join(stream)
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        self._collect_fetched()

    # ---- measurement helpers ------------------------------------------------------

    def resident_rows(self, t: int, stream=None) -> int:
        out = C.c_int64()
        _lib.check(self.lib.hc_engine_resident_rows(self.handle, t, C.byref(out),
                                                    _lib.stream_handle(stream)))
        return out.value

    PHASES = ("append", "attention", "combine", "score_rows", "monitor", "tail", "step",
              "inter_step_gap")

    def kernel_timing(self, enable: bool = True, light: bool = False) -> dict:
        """Summed device milliseconds per decode-step phase since the last call;
        then record every phase (enable), only the K4 attention phase (enable,
        light: two events per step) or nothing."""
        ms = (C.c_double * 8)()
        n = C.c_int32()
        level = (2 if light else 1) if enable else 0
        _lib.check(self.lib.hc_engine_timing(self.handle, level, ms, C.byref(n)))
        out = dict(zip(self.PHASES, list(ms)))
        out["steps"] = n.value
        return out

    def retrieval_stats(self) -> dict:
        """Host-link retrieval since the last call (needs kernel_timing enabled)."""
        out = (C.c_double * 4)()
        _lib.check(self.lib.hc_engine_retrieval_stats(self.handle, out))
        b, g, w, n = list(out)
        return {"bytes": b, "gather_ms": g, "landing_stall_ms": w, "batches": int(n),
                "host_link_gbs": (b / (g * 1e-3) / 1e9) if g > 0 else None}

    def prefill_stats(self) -> dict:
        out = (C.c_double * 3)()
        _lib.check(self.lib.hc_engine_prefill_stats(self.handle, out))
        return {"score_ms": out[0], "layers": int(out[1]), "window": int(out[2])}

    def active_tiles(self, t: int) -> int:
        n = C.c_int32()
        _lib.check(self.lib.hc_engine_active_tiles(self.handle, t, C.byref(n)))
        return n.value

    def pivot_row(self, b: int, p, t: int, dst, stream=None) -> None:
        _lib.check(self.lib.hc_engine_pivot_row(self.handle, self.unit(b, p), t, _lib.ptr(dst),
                                                _lib.stream_handle(stream)))

    def report(self, b: int, decode_steps: int, trace_sha256: str = "") -> SimulationReport:
        self.sync()
        st = self.states[b]
        return SimulationReport(policy=self.config.variant, trace_sha256=trace_sha256,
                                num_layers=self.NL, heads_per_layer=self.H, prefill_len=self.L,
                                decode_steps=decode_steps, budget_ceiling=self.plan.budget_ceiling,
                                update_delay_steps=self.config.update_delay_steps,
                                rows=tuple(st.rows), events=tuple(st.events))
