"""CPU oracle for the HeteroCache decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import it.  The product package (``paper_2601_13684_b200``) never imports it and
has no CPU fallback.

It is a plain numpy / pure-Python restatement of the reference algorithm
(``/root/reference/pkg/src/heterocache``), one function per reference routine,
each citing the file:line it follows.  It shares no code with the reference or
with the product.

Parity pinning: every function here is checked in ``tests/test_oracle.py``
against fixtures produced by running the reference itself in the build
container (``tests/golden/make_golden.py``): the reference's own
``golden_replay.json``, engine runs on the reference's synthetic traces
(the replay-equivalence and drift suites of ``test_acceptance.py`` /
``test_engine.py``), sparse/dense top-k known answers with forced ties, and
budget plans.  Decision logic (top-k sets, drift triggers, completion steps,
bytes, budgets) is pinned bit-exactly.  The fp32 attention restatement in
``attention_oracle.py`` has no reference implementation (the reference moves
index sets, never tensors) -- that part is "parity unpinned" against the
reference and is only a tolerance oracle.
"""

from __future__ import annotations

import statistics
from math import ceil, floor

import numpy as np

PAD_INDEX = 0xFFFFFFFF
FULL_ROLES = ("volatile", "pivot")
COMPRESSED_ROLES = ("anchor", "satellite")


# ---------------------------------------------------------------------------
# Selection: metrics.py:26-71
# ---------------------------------------------------------------------------


def top_k_sparse(indices, scores, k: int) -> np.ndarray:
    """Top-k of (index, score) candidates, PAD skipped; metrics.py:42-45.

    Order is score descending then index ascending; the comparison is on the
    float32 values promoted exactly to float64 (as Python's ``float()`` does).
    Returns the selected indices sorted ascending (a set in the reference).
    """
    idx = np.asarray(indices, dtype=np.uint64)
    sc = np.asarray(scores, dtype=np.float32).astype(np.float64)
    live = idx != PAD_INDEX
    idx, sc = idx[live], sc[live]
    if k <= 0 or idx.size == 0:
        return np.zeros(0, dtype=np.uint32)
    order = np.lexsort((idx, -sc))  # last key is primary
    return np.sort(idx[order[:k]]).astype(np.uint32)


def top_k_dense(weights, k: int, pool_kernel: int = 0) -> np.ndarray:
    """Dense top-k with optional zero-padded moving average; metrics.py:26-39.

    Order: pooled desc, raw desc, position asc.  Returns sorted positions.
    """
    w = np.asarray(weights, dtype=np.float64)
    if k <= 0:
        return np.zeros(0, dtype=np.uint32)
    if pool_kernel:
        if pool_kernel < 1 or pool_kernel % 2 == 0:
            raise ValueError("pool kernel must be odd and positive")
        pooled = np.convolve(w, np.ones(pool_kernel), mode="same") / pool_kernel
    else:
        pooled = w
    order = np.lexsort((np.arange(w.size), -w, -pooled))
    return np.sort(order[:k]).astype(np.uint32)


def top_k_dense_select(weights, k: int) -> np.ndarray:
    """top_k_dense(weights, k) (no pooling) in O(n): the k-th largest value by
    partition, every value above it, then the tied values in position order --
    the same set as the lexsort order (value desc, position asc), sorted.
    Rows holding NaN take the lexsort path."""
    w = np.asarray(weights, dtype=np.float64)
    n = w.size
    if k <= 0:
        return np.zeros(0, dtype=np.uint32)
    if k >= n:
        return np.arange(n, dtype=np.uint32)
    if np.isnan(w).any():
        return top_k_dense(w, k)
    thr = np.partition(w, n - k)[n - k]
    above = np.flatnonzero(w > thr)
    ties = np.flatnonzero(w == thr)
    sel = np.concatenate([above, ties[:k - above.size]])
    sel.sort()
    return sel.astype(np.uint32)


def overlap_coefficient(a, b) -> float:
    """metrics.py:74-79 -- |A&B| / min(|A|,|B|)."""
    sa, sb = set(int(x) for x in a), set(int(x) for x in b)
    if not sa or not sb:
        raise ValueError("overlap coefficient is undefined for empty index sets")
    return len(sa & sb) / min(len(sa), len(sb))


# ---------------------------------------------------------------------------
# Budget: budget.py:108-232
# ---------------------------------------------------------------------------


def round_half_up(x: float) -> int:
    """budget.py:108-110."""
    return floor(x + 0.5)


def base_length(rho, num_heads, num_full, num_comp, prefill_len) -> float:
    """Eq. 7, budget.py:113-125 (same float64 operation order)."""
    if num_comp <= 0:
        raise ValueError("no compressed heads to allocate")
    l_base = (rho * num_heads - num_full) * prefill_len / num_comp
    if l_base <= 0.0:
        raise ValueError("infeasible budget")
    return l_base


def _largest_remainder(shares, total):
    """budget.py:128-141: floors, then +1 by (floor - share, index) ascending."""
    floors = [floor(s) for s in shares]
    leftover = total - sum(floors)
    if leftover < 0 or leftover > len(shares):
        raise ValueError("share sum inconsistent with total")
    ranked = sorted(range(len(shares)), key=lambda i: (floors[i] - shares[i], i))
    out = list(floors)
    for i in ranked[:leftover]:
        out[i] += 1
    return out


def allocate(stabilities: dict, l_base: float, *, rho, epsilon, min_length,
             rounding, prefill_len, num_full) -> dict:
    """budget.py:144-208.  Returns a plan dict (lengths keyed by head id)."""
    heads = sorted(stabilities)
    n = len(heads)
    total = round_half_up(n * l_base)
    w = [1.0 / (stabilities[h] + epsilon) for h in heads]
    wsum = sum(w)
    shares = [total * x / wsum for x in w]
    lo = [i for i, s in enumerate(shares) if s < min_length]
    hi = [i for i, s in enumerate(shares) if s > prefill_len]
    if lo or hi:
        fixed = {i: min_length for i in lo}
        fixed.update({i: prefill_len for i in hi})
        free = [i for i in range(n) if i not in fixed]
        rest = max(0, total - sum(fixed.values()))
        if free:
            fw = sum(w[i] for i in free)
            fs = [rest * w[i] / fw for i in free]
            if rounding == "largest_remainder":
                fi = _largest_remainder(fs, rest)
            else:
                fi = [floor(s) for s in fs]
            ints = [0] * n
            for i, v in fixed.items():
                ints[i] = v
            for i, v in zip(free, fi):
                ints[i] = min(max(v, min_length), prefill_len)
        else:
            ints = [fixed[i] for i in range(n)]
    elif rounding == "largest_remainder":
        ints = _largest_remainder(shares, total)
    else:
        ints = [floor(s) for s in shares]
    return {
        "rho": rho, "prefill_len": prefill_len, "num_heads": num_full + n,
        "num_full": num_full, "num_comp": n, "l_base": l_base,
        "l_base_int": round_half_up(l_base),
        "lengths": {h: int(v) for h, v in zip(heads, ints)},
    }


def plan_budget(roles: dict, stabilities: dict, *, rho, prefill_len, epsilon=1e-6,
                min_length=16, rounding="largest_remainder") -> dict:
    """budget.py:211-232 given roles and per-head stability."""
    full = sorted(h for h, r in roles.items() if r in FULL_ROLES)
    comp = sorted(h for h, r in roles.items() if r in COMPRESSED_ROLES)
    l_base = base_length(rho, len(roles), len(full), len(comp), prefill_len)
    return allocate({h: stabilities[h] for h in comp}, l_base, rho=rho,
                    epsilon=epsilon, min_length=min_length, rounding=rounding,
                    prefill_len=prefill_len, num_full=len(full))


# ---------------------------------------------------------------------------
# Taxonomy: profiling.py:286-454, metrics.py:82-129
# ---------------------------------------------------------------------------


def _step_sets(indices, scores, k):
    """metrics.py:113-129: per (layer, head) list of per-step top-k sets."""
    T1, NL, H, _ = indices.shape
    return {
        (l, h): [frozenset(int(x) for x in top_k_sparse(indices[s, l, h], scores[s, l, h], k))
                 for s in range(T1)]
        for l in range(NL) for h in range(H)
    }


def run_taxonomy(traces, *, tau_stable=0.5, tau_sim=0.5, profiling_topk=None,
                 adjacency_step=None):
    """profile + build_adjacency + greedy_star_cluster + assign_roles.

    traces: list of (indices, scores, prefill_len).  Returns
    (roles, cluster_of, clusters, s_stable, s_sim) with clusters a list of
    (pivot, satellites tuple).
    """
    NL, H = traces[0][0].shape[1], traces[0][0].shape[2]
    heads = [(l, h) for l in range(NL) for h in range(H)]
    acc = {hd: [0.0, 0.0] for hd in heads}
    pair = {}
    for idx, sc, L in traces:
        k = profiling_topk if profiling_topk is not None else min(1000, ceil(L / 10))
        sets = _step_sets(idx, sc, k)
        T = idx.shape[0] - 1
        for (l, h) in heads:
            own = sets[(l, h)]
            stab = float(np.median([overlap_coefficient(s, own[0]) for s in own[1:]]))
            peers = [sets[(l, p)][1:] for p in range(H) if p != h]
            if peers:
                sim = float(np.median([max(overlap_coefficient(own[1:][t], p[t]) for p in peers)
                                       for t in range(T)]))
            else:
                sim = 0.0
            acc[(l, h)][0] += stab
            acc[(l, h)][1] += sim
        steps = [adjacency_step] if adjacency_step is not None else range(1, T + 1)
        for l in range(NL):
            for h1 in range(H):
                for h2 in range(h1 + 1, H):
                    vals = [overlap_coefficient(sets[(l, h1)][t], sets[(l, h2)][t]) for t in steps]
                    pair[(l, h1, h2)] = pair.get((l, h1, h2), 0.0) + float(np.median(vals))
    n = len(traces)
    s_stable = {hd: a[0] / n for hd, a in acc.items()}
    s_sim = {hd: a[1] / n for hd, a in acc.items()}
    adj = {hd: set() for hd in heads}
    for (l, h1, h2), tot in pair.items():
        if tot / n >= tau_sim:
            adj[(l, h1)].add((l, h2))
            adj[(l, h2)].add((l, h1))
    # greedy star clustering, profiling.py:370-394
    unassigned = set(heads)
    clusters = []
    while True:
        best, best_deg = None, 0
        for node in sorted(unassigned):
            deg = len((adj[node] & unassigned) - {node})
            if deg > best_deg:
                best, best_deg = node, deg
        if best is None:
            break
        sats = tuple(sorted((adj[best] & unassigned) - {best}))
        clusters.append((best, sats))
        unassigned -= {best, *sats}
    roles, cluster_of = {}, {}
    for cid, (p, sats) in enumerate(clusters):
        roles[p] = "pivot"
        cluster_of[p] = cid
        for s in sats:
            roles[s] = "satellite"
            cluster_of[s] = cid
    for hd in heads:
        if hd not in roles:
            roles[hd] = "anchor" if s_stable[hd] >= tau_stable else "volatile"
    return roles, cluster_of, clusters, s_stable, s_sim


# ---------------------------------------------------------------------------
# Engine replay: engine.py:52-425, evaluation.py:41-59
# ---------------------------------------------------------------------------


def resident_positions(L, t, base, sink_count, recency_window) -> set:
    """CacheView membership (engine.py:98-115) materialised as a set."""
    members = set(range(L, L + t))
    if base is None:
        members.update(range(L))
        return members
    members.update(range(min(sink_count, L)))
    members.update(range(max(0, L + t - recency_window), L))
    members.update(int(x) for x in base)
    return members


def cache_view_size(L, t, base, sink_count, recency_window) -> int:
    """engine.py:109-115."""
    if base is None:
        return L + t
    extras = set(range(min(sink_count, L)))
    extras.update(range(max(0, L + t - recency_window), L))
    return len(set(base) | extras) + t


def _recall(L, t, base, sink_count, recency_window, idx_row, sc_row) -> float:
    """evaluation.py:41-59 over engine.py:98-107 membership (sequential sums)."""
    total = 0.0
    hit = 0.0
    tail_floor = L + t - recency_window
    for i, s in zip(idx_row.tolist(), sc_row.tolist()):
        if i == PAD_INDEX:
            continue
        total += s
        if i >= L or base is None or i < sink_count or i >= tail_floor or i in base:
            hit += s
    if total == 0.0:
        return 1.0
    return hit / total


def replay(indices, scores, *, prefill_len, bytes_per_kv_entry, roles, clusters,
           lengths, l_base_int, tau_drift=0.5, window=8, transfer_bandwidth=1 << 30,
           update_delay_steps=1, sink_count=4, recency_window=8,
           variant="heterocache", eval_every_step=False, measure=True, record_dynamic=False):
    """Straight-line restatement of CacheEngine.run (engine.py:372-416).

    indices/scores: (T+1, NL, H, K) trace arrays (dense rows are K = L+T with
    PAD suffixes).  clusters: list of (pivot, satellites).  Returns a dict with
    rows (list of dicts mirroring StepRow), events (dicts mirroring
    RetrievalRecord) and final GPU sets.  measure=False skips the recall
    diagnostic (NaN) for traces that only carry pivot rows after step 0;
    record_dynamic=True also returns the dynamic sets in force at every step.
    """
    L = prefill_len
    T = indices.shape[0] - 1
    NL, H = indices.shape[1], indices.shape[2]
    heads = [(l, h) for l in range(NL) for h in range(H)]
    full = {hd for hd in heads if roles[hd] in FULL_ROLES}
    comp = sorted(hd for hd in heads if roles[hd] in COMPRESSED_ROLES)
    pivots = sorted(hd for hd in heads if roles[hd] == "pivot")
    sats_of = {p: tuple(s) for p, s in clusters}

    def eff_len(hd):  # engine.py:218-221
        return l_base_int if variant == "no_allocation" else lengths[hd]

    def top(step, hd, k):  # engine.py:229-230
        l, h = hd
        return frozenset(int(x) for x in top_k_sparse(indices[step, l, h], scores[step, l, h], k))

    def pivot_top(step, p):  # engine.py:232-240
        s = top(step, p, l_base_int)
        if len(s) < l_base_int:
            raise ValueError(f"pivot {p} has fewer than {l_base_int} live entries at {step}")
        return s

    # prefill_init, engine.py:263-274
    dynamic = {hd: top(0, hd, eff_len(hd)) for hd in comp}
    k_base, buffers = {}, {}
    if variant != "no_retrieval":
        for p in pivots:
            k_base[p] = pivot_top(0, p)
            buffers[p] = []
    pending = []  # (completion, order, satellite, frozenset)
    events = []
    cum = 0
    order = 0

    def measure_row(t):  # engine.py:276-288
        recs, total_size = [], 0
        for hd in heads:
            base = None if hd in full else dynamic[hd]
            l, h = hd
            if measure:
                recs.append(_recall(L, t, base, sink_count, recency_window,
                                    indices[t, l, h], scores[t, l, h]))
            total_size += cache_view_size(L, t, base, sink_count, recency_window)
        charged = len(full) * L + sum(len(dynamic[hd]) for hd in comp)
        recall = sum(recs) / len(recs) if measure else float("nan")
        return recall, charged, total_size - charged

    def in_flight(t):  # engine.py:140-143
        return sum(e["transfer_bytes"] for e in events if e["completion_step"] > t)

    dyn_trace = [dict(dynamic)] if record_dynamic else None
    r, c, x = measure_row(0)
    rows = [dict(step=0, recall=r, gpu_entries=c, extra_entries=x, bytes_in_flight=0,
                 cumulative_bytes=0, retrieval_flag=0)]
    for t in range(1, T + 1):  # decode_step, engine.py:290-370
        due = sorted((e for e in pending if e[0] <= t), key=lambda e: (e[0], e[1]))
        pending = [e for e in pending if e[0] > t]
        for _, _, s, ids in due:
            dynamic[s] = ids
        if record_dynamic:
            dyn_trace.append(dict(dynamic))
        r, c, x = measure_row(t)
        flag = 0
        if variant != "no_retrieval":
            cur = {}
            for p in pivots:
                cur[p] = pivot_top(t, p)
                buffers[p].append(len(cur[p] & k_base[p]) / l_base_int)
            for p in pivots:
                ready = len(buffers[p]) >= window if eval_every_step else t % window == 0
                if not ready:
                    continue
                vals = buffers[p][-window:]
                fired = bool(statistics.median(vals) < tau_drift)  # engine.py:247-250
                if fired:
                    flag = 1
                    fetches = []
                    n_ent = 0
                    for s in sats_of[p]:
                        got = top(t, p, eff_len(s))
                        fetches.append((s, tuple(sorted(got))))
                        n_ent += len(got)
                    nbytes = n_ent * bytes_per_kv_entry
                    cum += nbytes
                    completion = max(t + update_delay_steps, ceil(cum / transfer_bandwidth))
                    for s, ids in fetches:
                        pending.append((completion, order, s, frozenset(ids)))
                        order += 1
                    events.append(dict(trigger_step=t, pivot=p, completion_step=completion,
                                       transfer_bytes=nbytes, fetches=tuple(fetches)))
                    k_base[p] = cur[p]
                if fired or not eval_every_step:
                    buffers[p] = []
        rows.append(dict(step=t, recall=r, gpu_entries=c, extra_entries=x,
                         bytes_in_flight=in_flight(t), cumulative_bytes=cum,
                         retrieval_flag=flag))
    final = {hd: frozenset(resident_positions(L, T, None if hd in full else dynamic[hd],
                                              sink_count, recency_window)) for hd in heads}
    return {"rows": rows, "events": events, "final_gpu": final, "dynamic": dynamic,
            "k_base": k_base, "dynamic_trace": dyn_trace}


# ---- baseline policies (evaluation.py:60-228) --------------------------------


class PolicyError(ValueError):
    """evaluation.py:33-34 EvaluationError."""


def policy_window(rho, sink_count, window, prefill_len) -> int:
    """PolicySpec.effective_window (evaluation.py:85-94)."""
    if window is not None:
        return window
    w = floor(rho * prefill_len) - sink_count
    if w < 0:
        raise PolicyError("sink_count exceeds the budget")
    return w


def policy_budget_ceiling(name, rho, sink_count, window, num_heads, prefill_len) -> float:
    """PolicySpec.budget_ceiling (evaluation.py:96-102)."""
    if name == "full_oracle":
        return float(num_heads * prefill_len)
    if name == "sink_window":
        per_head = min(sink_count + policy_window(rho, sink_count, window, prefill_len),
                       prefill_len)
        return float(num_heads * per_head)
    return rho * num_heads * prefill_len


def static_policy_report(indices, scores, *, prefill_len, name, rho=0.5, sink_count=4,
                         window=None, engine_sink_count=4, engine_recency_window=8) -> dict:
    """run_policy for full_oracle / static_topk / sink_window (evaluation.py:165-228)
    through _static_rows (evaluation.py:110-162): per-head sets frozen for the
    whole decode.  Returns the SimulationReport fields that depend on the trace
    (rows, budget_ceiling, update_delay_steps, events)."""
    T1, NL, H, _ = indices.shape
    L = prefill_len
    heads = [(l, h) for l in range(NL) for h in range(H)]
    if name == "full_oracle":
        base, S, R = {hd: None for hd in heads}, 0, 0
    elif name == "static_topk":
        k = floor(rho * L)
        if k < 1:
            raise PolicyError("rho leaves no budget for static_topk")
        base = {(l, h): frozenset(int(x) for x in top_k_sparse(indices[0, l, h],
                                                               scores[0, l, h], k))
                for l, h in heads}
        S, R = engine_sink_count, engine_recency_window
    elif name == "sink_window":
        R = policy_window(rho, sink_count, window, L)
        base, S = {hd: frozenset() for hd in heads}, sink_count
    else:
        raise PolicyError(f"not a static policy: {name}")
    charged = sum(L if base[hd] is None else len(base[hd]) for hd in heads)
    rows = []
    for t in range(T1):
        recalls, total = [], 0
        for l, h in heads:
            b = base[(l, h)]
            recalls.append(_recall(L, t, b, S, R, indices[t, l, h], scores[t, l, h]))
            total += cache_view_size(L, t, b, S, R)
        rows.append(dict(step=t, recall=sum(recalls) / len(recalls), gpu_entries=charged,
                         extra_entries=total - charged, bytes_in_flight=0, cumulative_bytes=0,
                         retrieval_flag=0))
    return {"policy": name, "rows": rows, "events": [], "update_delay_steps": 0,
            "budget_ceiling": policy_budget_ceiling(name, rho, sink_count, window, len(heads), L)}
