"""Head profiling and role taxonomy (calibration; runs once, off the decode path).

Restates the reference taxonomy (profiling.py:43-454, metrics.py:74-129):
per-step top-k sets, stability (median overlap with the prefill set),
similarity (median of best same-step peer overlap), the same-layer agreement
graph (edge iff mean over traces of the median pair overlap >= tau_sim),
greedy star clustering (most unassigned neighbours, ties to the lowest
(layer, head)) and role assignment.

Device work: every (trace, step, layer, head) top-k set is selected by the
K1 kernel in one batched launch (the reference's per-row Python sort,
metrics.py:113-129), and every intersection size the overlap coefficients
need is an entry of a per-layer Gram matrix of the sets' 0/1 indicator
matrix, computed by K6 on the tcgen05 tensor cores (exact integer counts in
fp32).  Medians, the agreement graph and the clustering stay on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil
from typing import Optional

import numpy as np

ROLES = ("volatile", "anchor", "pivot", "satellite")
FULL_ROLES = ("volatile", "pivot")
COMPRESSED_ROLES = ("anchor", "satellite")


class TaxonomyError(ValueError):
    pass


@dataclass(frozen=True)
class ProfileConfig:
    tau_stable: float = 0.5
    tau_sim: float = 0.5
    profiling_topk: Optional[int] = None
    adjacency_step: Optional[int] = None

    def __post_init__(self):
        for name in ("tau_stable", "tau_sim"):
            v = getattr(self, name)
            if not (0.0 <= v <= 1.0):
                raise TaxonomyError(f"{name} must be in [0, 1], got {v}")
        if self.profiling_topk is not None and self.profiling_topk < 1:
            raise TaxonomyError(f"profiling_topk must be positive, got {self.profiling_topk}")

    def effective_topk(self, prefill_len: int) -> int:
        if self.profiling_topk is not None:
            return self.profiling_topk
        return min(1000, ceil(prefill_len / 10))  # metrics.py:109-110


@dataclass(frozen=True)
class HeadScores:
    s_stable: float
    s_sim: float


@dataclass(frozen=True)
class Cluster:
    cluster_id: int
    pivot: tuple
    satellites: tuple

    def members(self):
        return (self.pivot,) + tuple(self.satellites)


@dataclass(frozen=True)
class HeadProfile:
    layer: int
    head: int
    s_stable: float
    s_sim: float
    role: str
    cluster_id: Optional[int] = None

    def __post_init__(self):
        if self.role not in ROLES:
            raise TaxonomyError(f"unknown role {self.role!r}")
        if (self.role in ("pivot", "satellite")) != (self.cluster_id is not None):
            raise TaxonomyError(f"head ({self.layer}, {self.head}): role/cluster mismatch")

    @property
    def head_id(self):
        return (self.layer, self.head)


@dataclass(frozen=True)
class TaxonomyResult:
    num_layers: int
    heads_per_layer: int
    tau_stable: float
    tau_sim: float
    profiling_topk: Optional[int]
    heads: dict = field(hash=False)
    clusters: tuple = ()

    def role_counts(self) -> dict:
        counts = dict.fromkeys(ROLES, 0)
        for p in self.heads.values():
            counts[p.role] += 1
        return counts

    def _with_role(self, roles):
        return sorted(h for h, p in self.heads.items() if p.role in roles)

    def full_heads(self):
        return self._with_role(FULL_ROLES)

    def compressed_heads(self):
        return self._with_role(COMPRESSED_ROLES)

    def pivots(self):
        return self._with_role(("pivot",))

    def cluster_of(self, head_id):
        cid = self.heads[head_id].cluster_id
        return None if cid is None else self.clusters[cid]

    def to_json_dict(self) -> dict:
        return {
            "num_layers": self.num_layers, "heads_per_layer": self.heads_per_layer,
            "tau_stable": self.tau_stable, "tau_sim": self.tau_sim,
            "profiling_topk": self.profiling_topk,
            "heads": [{"layer": p.layer, "head": p.head, "s_stable": p.s_stable,
                       "s_sim": p.s_sim, "role": p.role, "cluster_id": p.cluster_id}
                      for _, p in sorted(self.heads.items())],
            "clusters": [{"cluster_id": c.cluster_id, "pivot": list(c.pivot),
                          "satellites": [list(s) for s in c.satellites]} for c in self.clusters],
            "role_counts": self.role_counts(),
        }

    @classmethod
    def from_json_dict(cls, p: dict) -> "TaxonomyResult":
        try:
            heads = {}
            for e in p["heads"]:
                hp = HeadProfile(layer=int(e["layer"]), head=int(e["head"]),
                                 s_stable=float(e["s_stable"]), s_sim=float(e["s_sim"]),
                                 role=str(e["role"]),
                                 cluster_id=None if e["cluster_id"] is None else int(e["cluster_id"]))
                heads[hp.head_id] = hp
            clusters = tuple(Cluster(int(c["cluster_id"]), tuple(int(x) for x in c["pivot"]),
                                     tuple(tuple(int(x) for x in s) for s in c["satellites"]))
                             for c in p["clusters"])
            res = cls(num_layers=int(p["num_layers"]), heads_per_layer=int(p["heads_per_layer"]),
                      tau_stable=float(p["tau_stable"]), tau_sim=float(p["tau_sim"]),
                      profiling_topk=None if p.get("profiling_topk") is None
                      else int(p["profiling_topk"]),
                      heads=heads, clusters=clusters)
        except TaxonomyError:
            raise
        except (KeyError, TypeError, ValueError) as exc:
            raise TaxonomyError(f"malformed taxonomy payload: {exc}") from exc
        res.validate()
        return res

    def validate(self) -> None:
        want = {(l, h) for l in range(self.num_layers) for h in range(self.heads_per_layer)}
        if set(self.heads) != want:
            raise TaxonomyError("taxonomy must cover every head exactly once")
        for i, c in enumerate(self.clusters):
            m = c.members()
            if c.cluster_id != i:
                raise TaxonomyError("cluster ids must be consecutive from zero")
            if len(set(m)) != len(m) or len(m) < 2:
                raise TaxonomyError(f"cluster {i} is degenerate")
            if len({l for l, _ in m}) != 1:
                raise TaxonomyError(f"cluster {i} spans layers")
            if self.heads[c.pivot].role != "pivot":
                raise TaxonomyError(f"cluster {i} pivot has a non-pivot role")
            for s in c.satellites:
                if self.heads[s].role != "satellite" or self.heads[s].cluster_id != i:
                    raise TaxonomyError(f"cluster {i} satellite {s} is inconsistent")
        for hd, p in self.heads.items():
            if p.cluster_id is not None:
                if p.cluster_id >= len(self.clusters) or hd not in self.clusters[p.cluster_id].members():
                    raise TaxonomyError(f"head {hd} is not in its own cluster")


def aggregate_gqa(query_scores, group_size: int) -> np.ndarray:
    """profiling.py:253-267: mean of consecutive query-head groups."""
    s = np.asarray(query_scores, dtype=np.float64)
    if s.ndim != 2:
        raise ValueError("expected a 2-D (heads, positions) array")
    if group_size < 1 or s.shape[0] % group_size:
        raise ValueError(f"group size {group_size} does not divide {s.shape[0]} query heads")
    return s.reshape(s.shape[0] // group_size, group_size, -1).mean(axis=1)


def step_set_gram(trace, k: int):
    """Per-layer intersection counts of all per-step top-k sets, on the GPU.

    K1 selects every (step, layer, head) top-k set in one batched launch
    (metrics.py:113-129); K6 forms the Gram matrix of the 0/1 indicator
    matrix of each layer's (step, head) sets on the tcgen05 tensor cores.
    Returns (gram [NL, S, S] int64 with S = (T+1)*H, set index t*H + h;
    sizes [T+1, NL, H]).
    """
    import torch

    from . import _lib
    from .ops import topk_rows

    idx = trace.indices
    T1, NL, H, K = idx.shape
    sel, cnt = topk_rows(idx.reshape(-1, K), trace.scores.reshape(-1, K), k)
    kk = sel.shape[1]
    sel = sel.reshape(T1, NL, H, kk).transpose(1, 0, 2, 3).reshape(NL, T1 * H, kk)
    cnt4 = cnt.reshape(T1, NL, H)
    sets = T1 * H
    rows_pad = (sets + 127) // 128 * 128
    d_sel = torch.from_numpy(np.ascontiguousarray(sel).view(np.int32)).cuda()
    d_cnt = torch.from_numpy(np.ascontiguousarray(cnt4.transpose(1, 0, 2).reshape(NL, sets))
                             .view(np.int32)).cuda()
    gram = torch.zeros((NL, rows_pad, rows_pad), dtype=torch.float32, device="cuda")
    n_pos = trace.manifest.prefill_len + trace.manifest.decode_steps
    _lib.check(_lib.load().hc_gram_from_sets(_lib.ptr(d_sel), _lib.ptr(d_cnt), NL, sets, kk,
                                             n_pos, _lib.ptr(gram), _lib.stream_handle()))
    g = gram.cpu().numpy()[:, :sets, :sets].astype(np.int64)
    return g, cnt4.astype(np.int64)


def _geometry(traces):
    if not traces:
        raise TaxonomyError("profiling requires at least one trace")
    m0 = traces[0].manifest
    for t in traces[1:]:
        if (t.manifest.num_layers, t.manifest.heads_per_layer) != (m0.num_layers, m0.heads_per_layer):
            from .trace import TraceInvariantError
            raise TraceInvariantError("calibration traces disagree on layer/head counts")
    return m0.num_layers, m0.heads_per_layer


def _profile_and_pairs(traces, config: ProfileConfig):
    """Stability / similarity scores and the agreement graph (profiling.py:286-367).

    Per trace, every intersection count comes from one Gram matrix per layer
    (step_set_gram, K1 + K6 on the GPU); the overlap coefficients, per-head
    medians over decode steps and the sums over traces are then numpy array
    operations with the reference's exact arithmetic: int / int in float64,
    np.median (same partition and middle-pair mean as the reference's
    per-list np.median), max over peers, and float64 accumulation in trace
    order.
    """
    NL, H = _geometry(traces)
    acc_st = np.zeros((NL, H))
    acc_sim = np.zeros((NL, H))
    pair = np.zeros((NL, H, H))
    empty = "overlap coefficient is undefined for empty index sets"
    for tr in traces:
        m = tr.manifest
        gram, size = step_set_gram(tr, config.effective_topk(m.prefill_len))
        T = m.decode_steps
        if T < 1:
            raise ValueError("stability requires at least one decode step")
        T1 = T + 1
        g = gram.reshape(NL, T1, H, T1, H)
        sz = size.transpose(1, 0, 2)  # [NL, T1, H]
        if (sz == 0).any():
            raise ValueError(empty)
        # stability: overlap of each decode-step set with the step-0 set (metrics.py:82-87)
        inter = np.stack([g[:, 1:, h, 0, h] for h in range(H)], axis=-1)  # [NL, T, H]
        den = np.minimum(sz[:, 1:, :], sz[:, :1, :])
        acc_st += np.median(inter.astype(np.float64) / den.astype(np.float64), axis=1)
        # same-step overlaps of every head pair: [NL, T1, H, H]
        tt = np.arange(T1)
        same = np.moveaxis(g[:, tt, :, tt, :], 0, 1).astype(np.float64)
        den2 = np.minimum(sz[:, :, :, None], sz[:, :, None, :]).astype(np.float64)
        ovp = same / den2
        if H > 1:  # similarity: best peer per step, median over steps (metrics.py:90-106)
            peers = ovp[:, 1:].copy()
            peers[:, :, np.arange(H), np.arange(H)] = -np.inf
            acc_sim += np.median(peers.max(axis=-1), axis=1)
        if config.adjacency_step is not None:
            if not 1 <= config.adjacency_step <= T:
                raise TaxonomyError(f"adjacency step {config.adjacency_step} outside 1..{T}")
            steps = [config.adjacency_step]
        else:
            steps = list(range(1, T + 1))
        pair += np.median(ovp[:, steps], axis=1)  # [NL, H, H], used for h1 < h2
    n = len(traces)
    scores = {(l, h): HeadScores(s_stable=float(acc_st[l, h]) / n,
                                 s_sim=float(acc_sim[l, h]) / n)
              for l in range(NL) for h in range(H)}
    adjacency = {(l, h): set() for l in range(NL) for h in range(H)}
    for l in range(NL):
        for h1 in range(H):
            for h2 in range(h1 + 1, H):
                if float(pair[l, h1, h2]) / n >= config.tau_sim:
                    adjacency[(l, h1)].add((l, h2))
                    adjacency[(l, h2)].add((l, h1))
    return scores, {hd: frozenset(v) for hd, v in adjacency.items()}


def profile(traces, config: ProfileConfig = ProfileConfig()) -> dict:
    return _profile_and_pairs(traces, config)[0]


def build_adjacency(traces, config: ProfileConfig = ProfileConfig()) -> dict:
    return _profile_and_pairs(traces, config)[1]


def greedy_star_cluster(adjacency: dict):
    left = set(adjacency)
    clusters = []
    while True:
        pick, deg = None, 0
        for node in sorted(left):
            d = len((adjacency[node] & left) - {node})
            if d > deg:
                pick, deg = node, d
        if pick is None:
            return tuple(clusters), sorted(left)
        sats = tuple(sorted((adjacency[pick] & left) - {pick}))
        clusters.append(Cluster(len(clusters), pick, sats))
        left -= {pick, *sats}


def assign_roles(scores, clusters, unclustered, config: ProfileConfig, *, num_layers,
                 heads_per_layer) -> TaxonomyResult:
    cid = {}
    for c in clusters:
        for m in c.members():
            cid[m] = c.cluster_id
    pivots = {c.pivot for c in clusters}
    heads = {}
    for hd, sc in scores.items():
        if hd in cid:
            role = "pivot" if hd in pivots else "satellite"
        else:
            role = "anchor" if sc.s_stable >= config.tau_stable else "volatile"
        heads[hd] = HeadProfile(layer=hd[0], head=hd[1], s_stable=sc.s_stable, s_sim=sc.s_sim,
                                role=role, cluster_id=cid.get(hd))
    res = TaxonomyResult(num_layers=num_layers, heads_per_layer=heads_per_layer,
                         tau_stable=config.tau_stable, tau_sim=config.tau_sim,
                         profiling_topk=config.profiling_topk, heads=heads,
                         clusters=tuple(clusters))
    res.validate()
    return res


def run_taxonomy(traces, config: ProfileConfig = ProfileConfig()) -> TaxonomyResult:
    NL, H = _geometry(traces)
    scores, adjacency = _profile_and_pairs(traces, config)
    clusters, rest = greedy_star_cluster(adjacency)
    return assign_roles(scores, clusters, rest, config, num_layers=NL, heads_per_layer=H)


def taxonomy_from_roles(roles: dict, clusters, *, num_layers: int, heads_per_layer: int,
                        s_stable: Optional[dict] = None) -> TaxonomyResult:
    """Build a TaxonomyResult from explicit roles (bench / tests)."""
    cl = tuple(Cluster(i, tuple(p), tuple(tuple(s) for s in sats))
               for i, (p, sats) in enumerate(clusters))
    cid = {m: c.cluster_id for c in cl for m in c.members()}
    heads = {hd: HeadProfile(layer=hd[0], head=hd[1],
                             s_stable=(s_stable or {}).get(hd, 0.5), s_sim=0.0, role=r,
                             cluster_id=cid.get(hd)) for hd, r in roles.items()}
    res = TaxonomyResult(num_layers=num_layers, heads_per_layer=heads_per_layer,
                         tau_stable=0.5, tau_sim=0.5, profiling_topk=None, heads=heads,
                         clusters=cl)
    res.validate()
    return res
