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
eval_every_step), where the overlap counts are read back.

StepRow.recall is NaN here: attention-mass recall is a trace-replay
diagnostic that needs every head's full attention (evaluation.py:41-59).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from math import ceil

import numpy as np

from . import _lib
from .engine import EngineConfig, EngineError, InfeasibleStateError, completion_step
from .reporting import RetrievalRecord, SimulationReport, StepRow

ROLE_CODE = {"volatile": 0, "anchor": 1, "pivot": 2, "satellite": 3}


@dataclass
class SequenceState:
    """Per-sequence mirror of CacheState (engine.py:126-143)."""

    step: int = 0
    buffers: dict = field(default_factory=dict)       # pivot -> overlap values
    pending: list = field(default_factory=list)       # (completion, order, satellite, tid)
    events: list = field(default_factory=list)        # RetrievalRecord
    cumulative_bytes: int = 0
    order: int = 0
    dyn_count: dict = field(default_factory=dict)     # compressed head -> |dynamic|
    dyn_sets: dict = field(default_factory=dict)      # compressed head -> sorted positions
    rows: list = field(default_factory=list)

    def bytes_in_flight(self, step: int) -> int:
        return sum(e.transfer_bytes for e in self.events if e.completion_step > step)


class HeteroCacheDecoder:
    def __init__(self, taxonomy, plan, config: EngineConfig = EngineConfig(), *, batch: int,
                 group: int, max_decode: int, head_dim: int = 128, chunk: int = 1024,
                 host_pool: bool = True, bytes_per_kv_entry: int | None = None,
                 track_sets: bool = True):
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
        desc = _lib.EngineDesc(batch=batch, num_layers=self.NL, kv_heads=self.H, group=group,
                               head_dim=head_dim, prefill_len=self.L, max_decode=max_decode,
                               sink_count=config.sink_count, recency_window=config.recency_window,
                               l_base_int=self.l_base_int, chunk=chunk, monitor=int(self.monitor),
                               host_pool=int(host_pool))
        h = C.c_void_p()
        _lib.check(self.lib.hc_engine_create(C.byref(desc), roles.ctypes.data, lengths.ctypes.data,
                                             cpiv.ctypes.data, C.byref(h)))
        self.handle = h
        info = (C.c_int64 * 4)()
        _lib.check(self.lib.hc_engine_info(self.handle, info))
        self.device_bytes, self.host_bytes, self.arena_rows, self.n_pivot_units = list(info)
        # pivot slot order == ascending unit order
        self.pivot_units = [self.unit(b, p) for b in range(self.B) for p in self.pivots] \
            if self.monitor else []
        self.pivot_units.sort()
        self.pivot_slot = {u: i for i, u in enumerate(self.pivot_units)}
        self.states = [SequenceState() for _ in range(self.B)]
        self._prefilled = set()

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
        """k, v: [B, H, L, D] bf16 device tensors; q_last: [B, H*G, D] bf16."""
        for t, shape in ((k, (self.B, self.H, self.L, self.D)), (v, (self.B, self.H, self.L, self.D)),
                         (q_last, (self.B, self.H * self.G, self.D))):
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
            for hd in self.comp:
                k = self.effective_length(hd)
                st.dyn_count[hd] = min(k, self.L)
                if self.track_sets:
                    st.dyn_sets[hd] = self.dynamic_set(b, hd)
            if self.monitor:
                for p in self.pivots:
                    st.buffers[p] = []
            st.rows.append(self._row(st, 0, 0))

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

    def _row(self, st: SequenceState, t: int, flag: int) -> StepRow:
        charged = len(self.full) * self.L + sum(st.dyn_count.values())
        if self.track_sets:
            total = len(self.full) * (self.L + t) + sum(self._size_of(st, hd, t) for hd in self.comp)
            extra = total - charged
        else:
            extra = -1
        return StepRow(step=t, recall=math.nan, gpu_entries=charged, extra_entries=extra,
                       bytes_in_flight=st.bytes_in_flight(t), cumulative_bytes=st.cumulative_bytes,
                       retrieval_flag=flag)

    def decode_step(self, t: int, q, k_new, v_new, out, stream=None, *, rows: bool = True):
        """q/out: [B, NL, H*G, D] bf16; k_new/v_new: [B, NL, H, D] bf16 (device)."""
        cfg = self.config
        sh = _lib.stream_handle(stream)
        # 1. land due transfers, per sequence in (completion, order) order
        for b, st in enumerate(self.states):
            due = sorted((x for x in st.pending if x[0] <= t), key=lambda x: (x[0], x[1]))
            if due:
                st.pending = [x for x in st.pending if x[0] > t]
                for _, _, s, tid, fetched in due:
                    _lib.check(self.lib.hc_engine_land(self.handle, tid, sh))
                    st.dyn_count[s] = len(fetched)
                    if self.track_sets:
                        st.dyn_sets[s] = fetched
            st.step = t
        # 2-4. append, attention, pivot rows, top-l_base + overlap counts
        _lib.check(self.lib.hc_engine_decode_step(self.handle, t, _lib.ptr(q), _lib.ptr(k_new),
                                                  _lib.ptr(v_new), _lib.ptr(out), sh))
        flags = [0] * self.B
        if self.monitor:
            boundary = cfg.eval_every_step or (t % cfg.window == 0)
            if boundary:
                first = t if cfg.eval_every_step else max(1, t - cfg.window + 1)
                self._decide(t, first, flags, stream)
        if rows:
            for b, st in enumerate(self.states):
                st.rows.append(self._row(st, t, flags[b]))
        return flags

    def _decide(self, t: int, first: int, flags: list, stream) -> None:
        """Window test and firing (engine.py:305-360) for every sequence."""
        cfg = self.config
        n = t - first + 1
        counts = np.empty((n, len(self.pivot_units)), dtype=np.int32)
        _lib.check(self.lib.hc_engine_overlaps(self.handle, first, t, counts.ctypes.data,
                                               _lib.stream_handle(stream)))
        for b, st in enumerate(self.states):
            for p in self.pivots:
                col = self.pivot_slot[self.unit(b, p)]
                st.buffers[p].extend(int(c) / self.l_base_int for c in counts[:, col])
            for p in self.pivots:
                if cfg.eval_every_step:
                    ready = len(st.buffers[p]) >= cfg.window
                else:
                    ready = t % cfg.window == 0
                if not ready:
                    continue
                fired = bool(np.median(st.buffers[p][-cfg.window:]) < cfg.tau_drift)
                if fired:
                    flags[b] = 1
                    self._fire(b, st, p, t, stream)
                if fired or not cfg.eval_every_step:
                    st.buffers[p] = []

    def _fire(self, b: int, st: SequenceState, p, t: int, stream) -> None:
        sats = self.satellites_of[p]
        ks = [min(self.effective_length(s), self.L + t) for s in sats]
        nbytes = sum(ks) * self.bytes_per_entry
        st.cumulative_bytes += nbytes
        done = completion_step(t, st.cumulative_bytes, self.config)
        ids = np.zeros(len(sats), dtype=np.int32)
        _lib.check(self.lib.hc_engine_fire(self.handle, self.unit(b, p), t, done, ids.ctypes.data,
                                           _lib.stream_handle(stream)))
        fetches = []
        for s, k, tid in zip(sats, ks, ids.tolist()):
            got = self.read_indices(0, tid, k, stream)
            fetches.append((s, tuple(int(x) for x in got)))
            st.pending.append((done, st.order, s, tid, got))
            st.order += 1
        st.events.append(RetrievalRecord(trigger_step=t, pivot=p, completion_step=done,
                                         transfer_bytes=nbytes, fetches=tuple(fetches)))

    # ---- measurement helpers ------------------------------------------------------

    def resident_rows(self, t: int, stream=None) -> int:
        out = C.c_int64()
        _lib.check(self.lib.hc_engine_resident_rows(self.handle, t, C.byref(out),
                                                    _lib.stream_handle(stream)))
        return out.value

    def active_tiles(self, t: int) -> int:
        n = C.c_int32()
        _lib.check(self.lib.hc_engine_active_tiles(self.handle, t, C.byref(n)))
        return n.value

    def pivot_row(self, b: int, p, t: int, dst, stream=None) -> None:
        _lib.check(self.lib.hc_engine_pivot_row(self.handle, self.unit(b, p), t, _lib.ptr(dst),
                                                _lib.stream_handle(stream)))

    def report(self, b: int, decode_steps: int, trace_sha256: str = "") -> SimulationReport:
        st = self.states[b]
        return SimulationReport(policy=self.config.variant, trace_sha256=trace_sha256,
                                num_layers=self.NL, heads_per_layer=self.H, prefill_len=self.L,
                                decode_steps=decode_steps, budget_ceiling=self.plan.budget_ceiling,
                                update_delay_steps=self.config.update_delay_steps,
                                rows=tuple(st.rows), events=tuple(st.events))
