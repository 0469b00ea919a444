"""CPU decoder oracle -- TEST / BASELINE INFRASTRUCTURE ONLY.

A straight restatement, over real K/V tensors, of what the reference engine
does for ONE sequence (engine.py:263-370), with the attention semantics of the
exporter (model.ts:232-291) in fp32 on the host cores:

  prefill(layer, K, V, q_obs)   prefill_init (engine.py:263-274): step-0 rows =
                                the GQA-mean softmax row of the last prompt
                                token(s) (export.ts:125-127; w > 1: the mean of
                                the last w tokens' causal rows, as K5 computes);
                                dynamic_h = top_{l_h}, K_base = top_{l_base_int}
  step(t, q, k_new, v_new)      decode_step (engine.py:290-370): land due
                                transfers in (completion, order) order; every
                                head's attention over its CacheView resident set
                                (engine.py:98-115); pivot rows -> top_{l_base}
                                -> overlap with K_base (Eq. 9); at a window
                                boundary the median test, fetch selection
                                top_{l_s}(pivot row), byte / completion
                                accounting, K_base <- current top (engine.py:
                                313-357)

Selection is hc_oracle.top_k_dense's order (metrics.py:26-45), through its
O(n) twin top_k_dense_select (identical output, tested).  K / V are kept as fp32
copies of the bf16 inputs (exact), so a step reads each resident row once
instead of converting whole caches.  The decision
logic is the same sequence of operations as hc_oracle.replay (pinned to the
reference's own runs); only the rows come from this module's fp32 attention
instead of a trace.

Used by bench.py's reference arm / cpu_baseline leg (timed, on the same
seeded inputs as the GPU arm) and by tests/.  Never by the product path.
"""

from __future__ import annotations

import math
import statistics

import numpy as np
import torch

from . import hc_oracle as O


class CpuDecoder:
    def __init__(self, *, roles: dict, clusters, lengths: dict, l_base_int: int, prefill_len: int,
                 max_decode: int, group: int, head_dim: int = 128, tau_drift: float = 0.5,
                 window: int = 8, transfer_bandwidth: int = 1 << 30, update_delay_steps: int = 1,
                 sink_count: int = 4, recency_window: int = 8, bytes_per_kv_entry: int = 512,
                 variant: str = "heterocache", record_rows: bool = False):
        self.roles = dict(roles)
        self.record = {} if record_rows else None  # (t, pivot) -> row (tests)
        self.NL = 1 + max(l for l, _ in roles)
        self.H = 1 + max(h for _, h in roles)
        self.G, self.D, self.L, self.T = group, head_dim, prefill_len, max_decode
        self.sats_of = {tuple(p): tuple(tuple(s) for s in sats) for p, sats in clusters}
        self.lengths = dict(lengths)
        self.l_base = l_base_int
        self.tau, self.W = tau_drift, window
        self.bw, self.delay = transfer_bandwidth, update_delay_steps
        self.S, self.R, self.bpe = sink_count, recency_window, bytes_per_kv_entry
        self.variant = variant
        self.full = {hd for hd, r in roles.items() if r in ("volatile", "pivot")}
        self.comp = sorted(hd for hd, r in roles.items() if r in ("anchor", "satellite"))
        self.pivots = sorted(hd for hd, r in roles.items() if r == "pivot")
        self.monitor = bool(self.pivots) and variant != "no_retrieval"
        self.K, self.V = {}, {}
        self.dynamic, self.k_base, self.buffers = {}, {}, {}
        self.pending, self.events = [], []
        self.cum, self.order = 0, 0
        self.rows0 = {}
        self._base = {}  # hd -> (dynamic array, recency start, sorted positions < L)
        self._gath = {}  # hd -> (dynamic, recency start, K rows, V rows, rows < L, steps)

    def eff_len(self, hd) -> int:  # engine.py:218-221
        return self.l_base if self.variant == "no_allocation" else self.lengths[hd]

    # ---- prefill (engine.py:263-274) ------------------------------------------

    def prefill(self, layer: int, k, v, q_obs) -> None:
        """k, v [H, L, D] bf16; q_obs [H*G, D] (window 1) or [w, H*G, D]."""
        L, G, D = self.L, self.G, self.D
        q = q_obs if q_obs.dim() == 3 else q_obs[None]
        w = q.shape[0]
        for h in range(self.H):
            hd = (layer, h)
            kb = torch.empty(L + self.T, D, dtype=torch.float32)  # bf16 values, exact
            vb = torch.empty(L + self.T, D, dtype=torch.float32)
            kb[:L], vb[:L] = k[h], v[h]
            self.K[hd], self.V[hd] = kb, vb
            kf = kb[:L]
            acc = torch.zeros(L, dtype=torch.float32)
            for i in range(w):  # query i sits at prompt position L - w + i (causal)
                lim = L - w + i + 1
                s = (q[i, h * G:(h + 1) * G].float() @ kf[:lim].T) * (1.0 / math.sqrt(D))
                p = torch.softmax(s, dim=-1)
                acc[:lim] += p.sum(0)
            row = (acc / (w * G)).numpy()
            self.rows0[hd] = row
            if hd in self.comp:
                self.dynamic[hd] = O.top_k_dense_select(row, self.eff_len(hd))
            elif hd in self.pivots and self.monitor:
                self.k_base[hd] = O.top_k_dense_select(row, self.l_base)
                self.buffers[hd] = []

    # ---- decode (engine.py:290-370) ---------------------------------------------

    def resident(self, hd, t) -> np.ndarray | None:
        """Sorted CacheView positions of a compressed head at step t (None: full)."""
        if hd in self.full:
            return None
        L = self.L
        dyn, r0 = self.dynamic[hd], min(L, max(0, L + t - self.R))
        base = self._base.get(hd)
        if base is None or base[0] is not dyn or base[1] != r0:
            # dynamic | sinks | recency tail below L (union1d sorts); a fetched set
            # may hold decode positions >= L, which the appends [L, L + t) cover
            extra = np.concatenate([np.arange(min(self.S, L)), np.arange(r0, L)]).astype(np.int64)
            d64 = dyn.astype(np.int64)
            base = (dyn, r0, np.union1d(d64[d64 < L], extra))
            self._base[hd] = base
        return np.concatenate([base[2], np.arange(L, L + t, dtype=np.int64)])  # decode appends

    def resident_kv(self, hd, t):
        """K, V rows of head hd's resident set at step t, in position order (views).

        Full heads: the cache prefix.  Compressed heads: the rows below L (dynamic |
        sinks | recency tail) gathered once per change of that set into a per-head
        buffer, then the decode appends [L, L + t) -- the same rows in the same
        order as indexing the cache with resident(hd, t)."""
        L = self.L
        if hd in self.full:
            return self.K[hd][:L + t], self.V[hd][:L + t]
        dyn, r0 = self.dynamic[hd], min(L, max(0, L + t - self.R))
        g = self._gath.get(hd)
        if g is None or g[0] is not dyn or g[1] != r0:
            self.resident(hd, t)  # (re)computes the sorted positions below L
            base = self._base[hd][2]
            n0 = base.size
            kb = torch.empty(n0 + self.T, self.D, dtype=torch.float32)
            vb = torch.empty(n0 + self.T, self.D, dtype=torch.float32)
            ix = torch.from_numpy(base)
            torch.index_select(self.K[hd], 0, ix, out=kb[:n0])
            torch.index_select(self.V[hd], 0, ix, out=vb[:n0])
            kb[n0:n0 + t] = self.K[hd][L:L + t]
            vb[n0:n0 + t] = self.V[hd][L:L + t]
            g = (dyn, r0, kb, vb, n0, t)
        else:
            n0, kb, vb = g[4], g[2], g[3]
            if g[5] < t:  # the appends since the buffer was last used
                kb[n0 + g[5]:n0 + t] = self.K[hd][L + g[5]:L + t]
                vb[n0 + g[5]:n0 + t] = self.V[hd][L + g[5]:L + t]
            g = (dyn, r0, kb, vb, n0, t)
        self._gath[hd] = g
        return kb[:n0 + t], vb[:n0 + t]

    def step(self, t: int, q, k_new, v_new):
        """q [NL, H*G, D], k_new / v_new [NL, H, D] (bf16).  Returns (O [NL, H*G, D]
        fp32, retrieval flag)."""
        L, G = self.L, self.G
        due = sorted((e for e in self.pending if e[0] <= t), key=lambda e: (e[0], e[1]))
        self.pending = [e for e in self.pending if e[0] > t]
        for _, _, s, ids in due:  # engine.py:293-299
            self.dynamic[s] = ids
        out = torch.empty(self.NL, self.H * G, self.D, dtype=torch.float32)
        rows = {}
        for l in range(self.NL):
            for h in range(self.H):
                hd = (l, h)
                self.K[hd][L + t - 1] = k_new[l, h]
                self.V[hd][L + t - 1] = v_new[l, h]
                qh = q[l, h * G:(h + 1) * G].float()
                kk, vv = self.resident_kv(hd, t)
                s = (qh @ kk.T) * (1.0 / math.sqrt(self.D))
                s = s - s.max(dim=-1, keepdim=True).values
                e = torch.exp(s)
                p = e * (1.0 / e.sum(dim=-1, keepdim=True))
                out[l, h * G:(h + 1) * G] = p @ vv
                if hd in self.pivots and self.monitor:
                    acc = p[0].clone()
                    for j in range(1, G):  # GQA mean in head order (model.ts:283-289)
                        acc = acc + p[j]
                    rows[hd] = (acc / G).numpy()
                    if self.record is not None:
                        self.record[(t, hd)] = rows[hd]
        flag = 0
        if self.monitor:
            cur = {}
            for pv in self.pivots:
                cur[pv] = O.top_k_dense_select(rows[pv], self.l_base)
                self.buffers[pv].append(
                    np.intersect1d(cur[pv], self.k_base[pv], assume_unique=True).size / self.l_base)
            if t % self.W == 0:
                for pv in self.pivots:
                    vals = self.buffers[pv][-self.W:]
                    if statistics.median(vals) < self.tau:  # engine.py:247-250
                        flag = 1
                        fetches, n_ent = [], 0
                        for s in self.sats_of[pv]:  # engine.py:326-329
                            got = O.top_k_dense_select(rows[pv], min(self.eff_len(s), L + t))
                            fetches.append((s, tuple(int(x) for x in got)))
                            n_ent += len(got)
                        nbytes = n_ent * self.bpe
                        self.cum += nbytes
                        completion = max(t + self.delay, math.ceil(self.cum / self.bw))
                        for s, ids in fetches:
                            self.pending.append((completion, self.order, s,
                                                 np.asarray(ids, dtype=np.uint32)))
                            self.order += 1
                        self.events.append(dict(trigger_step=t, pivot=pv,
                                                completion_step=completion,
                                                transfer_bytes=nbytes, fetches=tuple(fetches)))
                        self.k_base[pv] = cur[pv]
                    self.buffers[pv] = []
        return out, flag
