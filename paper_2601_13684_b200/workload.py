"""Synthetic decode workloads: model shapes, head roles,
budgets and seeded bf16 K/V/Q with planted hot sets and topic shifts.

Noise is a counter-based generator (csrc/synth.cu on the GPU, so 128K-224K
contexts never touch host memory; a bit-identical host twin for the CPU
arms).  Roles per layer follow the survey's synthetic mix:
Llama-shaped layers hold 1 pivot + 4 satellites + 2 anchors + 1 volatile
head, Qwen-shaped layers 1 pivot + 2 satellites + 1 anchor.  "c% budget" is
read as L_base = c*L, i.e. rho = (N_full + c*N_comp) / N (SURVEY.md section 7,
hard part 6).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .budget import BudgetConfig, plan_budget
from .profiling import taxonomy_from_roles

LLAMA_LAYER = ("pivot", "satellite", "satellite", "satellite", "satellite", "anchor", "anchor",
               "volatile")
QWEN_LAYER = ("pivot", "satellite", "satellite", "anchor")


@dataclass(frozen=True)
class ModelShape:
    name: str
    num_layers: int
    q_heads: int
    kv_heads: int
    head_dim: int = 128

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads

    def layer_roles(self):
        return LLAMA_LAYER if self.kv_heads == 8 else QWEN_LAYER


LLAMA3_8B = ModelShape("Llama-3.1-8B", 32, 32, 8)
QWEN25_7B = ModelShape("Qwen2.5-7B", 28, 28, 4)
R1_LLAMA_8B = ModelShape("DeepSeek-R1-Distill-Llama-8B", 32, 32, 8)


@dataclass(frozen=True)
class Workload:
    name: str
    model: ModelShape
    prefill_len: int
    batch: int
    compression: float   # c: L_base = c * L
    decode_steps: int
    shift_every: int     # planted topic shift period (steps); 0 = DRIFT_PERIOD
    layers: int | None = None  # override (bench subsets); None = all layers
    # EngineConfig.transfer_bandwidth of timing runs ("set from the
    # measured host link"): the B200 box's measured link (~48 GB/s, zero-copy
    # gather) times the workload's measured decode step, in MiB per step
    link_mib_per_step: float = 64.0

    @property
    def num_layers(self) -> int:
        return self.layers or self.model.num_layers


# BASELINE.json configs
CONFIGS = {
    # link MiB/step = 48 GB/s x step: cfg1 0.05 ms, cfg2 0.27, cfg3 1.41, cfg4 0.57, cfg5 11.6
    "cfg1": Workload("llama3-8b-layer-4k-b1", LLAMA3_8B, 4096, 1, 0.10, 64, 0, layers=1,
                     link_mib_per_step=2.0),
    "cfg2": Workload("llama3.1-8b-32k-b1", LLAMA3_8B, 32768, 1, 0.10, 256, 0,
                     link_mib_per_step=12.0),
    "cfg3": Workload("qwen2.5-7b-128k-b4", QWEN25_7B, 131072, 4, 0.05, 128, 0,
                     link_mib_per_step=64.0),
    "cfg4": Workload("r1-distill-llama-8b-64k+8k-b1", R1_LLAMA_8B, 65536, 1, 0.10, 8192, 12,
                     link_mib_per_step=26.0),
    "cfg5": Workload("llama3.1-8b-224k-b8", LLAMA3_8B, 229376, 8, 0.10, 64, 0,
                     link_mib_per_step=530.0),
}


def roles_for(model: ModelShape, num_layers: int):
    """Taxonomy with the survey's role mix (one cluster per layer)."""
    per = model.layer_roles()
    roles = {(l, h): r for l in range(num_layers) for h, r in enumerate(per)}
    clusters = [((l, 0), [(l, h) for h, r in enumerate(per) if r == "satellite"])
                for l in range(num_layers)]
    # stabilities in [0.3, 0.8]: anchors steadier than satellites (inverse weighting)
    stab = {}
    for (l, h), r in roles.items():
        stab[(l, h)] = 0.75 if r == "anchor" else 0.45 + 0.05 * (h % 3)
    return taxonomy_from_roles(roles, clusters, num_layers=num_layers,
                               heads_per_layer=model.kv_heads, s_stable=stab)


def rho_for(model: ModelShape, c: float) -> float:
    per = model.layer_roles()
    n_full = sum(r in ("pivot", "volatile") for r in per)
    return (n_full + c * (len(per) - n_full)) / len(per)


def plan_for(w: Workload, policy: str = "heterocache"):
    """Taxonomy + plan of a workload.  policy "full" is the FullAttention
    baseline (evaluation.py:165-190 full_oracle): every head keeps its whole
    cache, nothing is monitored or retrieved."""
    if policy == "full":
        from .budget import BudgetPlan

        per = w.model.layer_roles()
        roles = {(l, h): "volatile" for l in range(w.num_layers) for h in range(len(per))}
        tax = taxonomy_from_roles(roles, [], num_layers=w.num_layers,
                                  heads_per_layer=w.model.kv_heads)
        plan = BudgetPlan(rho=1.0, prefill_len=w.prefill_len, num_heads=len(roles),
                          num_full=len(roles), num_comp=0, l_base=float(w.prefill_len),
                          l_base_int=w.prefill_len, lengths={})
        return tax, plan
    tax = roles_for(w.model, w.num_layers)
    plan = plan_budget(tax, BudgetConfig(rho=rho_for(w.model, w.compression), min_length=16),
                       w.prefill_len)
    return tax, plan


M64 = (1 << 64) - 1


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def stream_key(*parts: int) -> int:
    """64-bit key of one generator stream (seed, tensor kind, indices...)."""
    h = 0x6A09E667F3BCC908
    for p in parts:
        h = _splitmix64(h ^ (int(p) & M64))
    return h


class DeviceNormal:
    """N(key, offset + i) on the GPU (csrc/synth.cu, hc_synth_normal)."""

    device = "cuda"

    def __call__(self, shape, key: int, offset: int = 0):
        import torch

        from . import _lib

        out = torch.empty(shape, dtype=torch.float32, device="cuda")
        _lib.check(_lib.load().hc_synth_normal(out.data_ptr(), out.numel(), key & M64, offset,
                                               _lib.stream_handle()))
        return out


# generator stream kinds
_K, _V, _Q, _QN, _KN, _VN = 1, 2, 3, 4, 5, 6


class SyntheticKV:
    """Seeded K/V/Q with planted per-cluster hot sets and topic shifts.

    For each (sequence b, layer l) the cluster (pivot + satellites) shares two
    topic directions u0/u1 with hot position sets H0/H1; anchors own a fixed
    topic; the volatile head attends diffusely.  Keys at hot positions get
    +alpha*u, queries are beta*u(t) + N(0, I) with the cluster topic switching
    from u0 to u1 at the shift step, so the pivot's top set moves and the drift
    monitor fires (engine.py:313-321).

    Noise comes from a counter-based generator keyed by (seed, tensor, b, l,
    h): `normal` is the GPU generator by default; the CPU arms of the bench
    pass its bit-identical host twin (oracle/synth.py) and, with `seqs`,
    generate any subset of the batch's sequences -- the same values the GPU
    arm decodes.  Topic directions and hot sets come from a seeded CPU torch
    generator (identical on every host).
    """

    def __init__(self, model: ModelShape, *, batch: int, prefill_len: int, num_layers: int,
                 hot: int, seed: int, alpha: float = 9.0, beta: float = 9.0, device="cuda",
                 normal=None, seqs=None):
        import torch

        self.torch = torch
        self.m, self.B, self.L, self.NL = model, batch, prefill_len, num_layers
        self.D, self.H, self.G = model.head_dim, model.kv_heads, model.group
        self.hot, self.seed, self.alpha, self.beta = hot, seed, alpha, beta
        self.normal = normal or DeviceNormal()
        self.dev = getattr(self.normal, "device", device)
        self.seqs = list(range(batch)) if seqs is None else list(seqs)
        self.roles = model.layer_roles()
        self.n_anchor = sum(r == "anchor" for r in self.roles)
        nt = 2 + self.n_anchor
        g = torch.Generator(device="cpu").manual_seed(seed)
        # per (b, l): topic directions [B, NL, topics, D]: 0/1 the cluster's two
        # topics, 2 + a the a-th anchor's own steady topic (distinct anchors are
        # stable but not similar: profiling keeps them anchors, profiling.py:397-438)
        u = torch.randn(batch, num_layers, nt, self.D, generator=g)
        u = u / u.norm(dim=-1, keepdim=True)
        hot = min(hot, prefill_len // nt)
        hs = torch.stack([
            torch.stack([torch.randperm(prefill_len, generator=g)[:nt * hot].view(nt, hot)
                         for _ in range(num_layers)]) for _ in range(batch)])
        sel = torch.as_tensor(self.seqs, dtype=torch.long)
        self.u_all = u.to(self.dev)                 # every sequence (queries are batch-wide)
        self.u = u[sel].to(self.dev)                # the generated sequences
        self.hot_sets = hs[sel].to(self.dev)

    def _head_topic(self, h: int) -> int:
        """0: cluster head (topic 0/1), 2 + a: the a-th anchor, -1: volatile."""
        r = self.roles[h]
        if r == "anchor":
            return 2 + sum(x == "anchor" for x in self.roles[:h])
        return {"pivot": 0, "satellite": 0, "volatile": -1}[r]

    def layer_kv(self, layer: int, window: int = 1):
        """K, V [b, H, L, D] bf16 (b = the generated sequences) and the prefill
        observation queries for one layer: q_last [b, H*G, D] (window 1) or
        [b, window, H*G, D] (last `window` tokens)."""
        torch = self.torch
        H, L, D = self.H, self.L, self.D
        nb = len(self.seqs)
        k = torch.empty(nb, H, L, D, device=self.dev, dtype=torch.float32)
        v = torch.empty_like(k)
        for i, b in enumerate(self.seqs):
            for h in range(H):
                k[i, h] = self.normal((L, D), stream_key(self.seed, _K, b, layer, h))
                v[i, h] = self.normal((L, D), stream_key(self.seed, _V, b, layer, h))
        for h in range(H):
            tp = self._head_topic(h)
            if tp < 0:
                continue
            for topic in ((0, 1) if tp == 0 else (tp,)):
                idx = self.hot_sets[:, layer, topic]                      # [b, hot]
                add = self.alpha * self.u[:, layer, topic]               # [b, D]
                k[:, h].scatter_add_(1, idx[:, :, None].expand(-1, -1, D),
                                     add[:, None, :].expand(-1, idx.shape[1], -1).contiguous())
        if window == 1:
            q = self.queries(layer, 0)
        else:
            q = torch.stack([self.queries(layer, -1 - i) for i in range(window)][::-1], dim=1)
        return k.to(torch.bfloat16).contiguous(), v.to(torch.bfloat16).contiguous(), q.contiguous()

    def queries(self, layer: int, step: int, shift_step=None):
        """[b, H*G, D] bf16 queries of one layer at a decode step.  shift_step: the
        step of the planted topic shift, or a sequence of shift steps (the cluster
        topic toggles at each)."""
        torch = self.torch
        B, H, G, D = self.B, self.H, self.G, self.D
        q = self.normal((B, H, G, D), stream_key(self.seed, _Q, layer, step))
        for h in range(H):
            tp = self._head_topic(h)
            if tp < 0:
                continue
            if tp == 0 and shift_step is not None:
                shifts = shift_step if isinstance(shift_step, (list, tuple)) else (shift_step,)
                tp = sum(step >= x for x in shifts) % 2
            q[:, h] += self.beta * self.u_all[:, layer, tp][:, None, :]
        q = q[torch.as_tensor(self.seqs, device=q.device)] if len(self.seqs) != B else q
        return q.reshape(-1, H * G, D).to(torch.bfloat16).contiguous()

    def step_inputs(self, step: int, shift_step: int | None):
        """q [b, NL, H*G, D], k_new/v_new [b, NL, H, D] (bf16)."""
        torch = self.torch
        q = torch.stack([self.queries(l, step, shift_step) for l in range(self.NL)], dim=1)
        shp = (self.B, self.NL, self.H, self.D)
        kn = self.normal(shp, stream_key(self.seed, _KN, step))
        vn = self.normal(shp, stream_key(self.seed, _VN, step))
        sel = torch.as_tensor(self.seqs, device=kn.device)
        if len(self.seqs) != self.B:
            kn, vn = kn[sel], vn[sel]
        return (q.contiguous(), kn.to(torch.bfloat16).contiguous(),
                vn.to(torch.bfloat16).contiguous())


DRIFT_PERIOD = 300  # steps between a cluster's topic shifts (one per run)


def staggered_shifts(batch: int, num_layers: int, start: int, span: int, every: int = 0):
    """Per-(sequence, layer) cluster shift steps over [start, start + span).

    Every cluster's topic shifts once per `every` steps (0: DRIFT_PERIOD, the
    survey's "one shift per run" of 300 steps; cfg4: every 12 steps), with the
    clusters' phases spread evenly over the period.  The drift rate per step
    is therefore fixed by the workload, not by the length of the timed loop.
    Returns {(b, l): [steps]}.
    """
    every = every or DRIFT_PERIOD
    n = batch * num_layers
    out = {}
    for b in range(batch):
        for l in range(num_layers):
            i = b * num_layers + l
            out[(b, l)] = list(range(start + (i * every) // n, start + span, every))
    return out


def decode_queries(gen: "SyntheticKV", steps: int, shifts: dict, n_noise: int = 4):
    """Queries for decode steps 1..steps: [steps + 1, b, NL, H*G, D] bf16 (the
    generator's device; b = its generated sequences).

    Cluster heads (pivot, satellites) of (b, l) follow topic u0 or u1, toggling at
    each of that cluster's shift steps; noise cycles through n_noise draws."""
    torch = gen.torch
    B, NL, H, G, D = gen.B, gen.NL, gen.H, gen.G, gen.D
    sel = torch.as_tensor(gen.seqs, dtype=torch.long)
    nb = len(gen.seqs)
    noise = [gen.normal((B, NL, H, G, D), stream_key(gen.seed, _QN, i))[sel.to(gen.dev)]
             for i in range(n_noise)]
    cluster = torch.tensor([gen._head_topic(h) == 0 for h in range(H)], device=gen.dev)
    anchors = [(h, gen._head_topic(h)) for h in range(H) if gen._head_topic(h) >= 2]
    u = gen.u  # [b, NL, 3, D]
    out = torch.empty(steps + 1, nb, NL, H * G, D, device=gen.dev, dtype=torch.bfloat16)
    topic = torch.zeros(steps + 1, nb, NL, dtype=torch.long, device=gen.dev)
    for i, b in enumerate(gen.seqs):
        for l in range(NL):
            for x in shifts.get((b, l), ()):
                if 0 <= x <= steps:
                    topic[x:, i, l] ^= 1
    for t in range(steps + 1):
        ut = torch.gather(u, 2, topic[t][:, :, None, None].expand(nb, NL, 1, D))[:, :, 0]
        q = noise[t % n_noise].clone()
        q += gen.beta * (cluster[None, None, :, None, None] * ut[:, :, None, None, :])
        for h, tp in anchors:
            q[:, :, h] += gen.beta * u[:, :, tp][:, :, None, :]
        out[t] = q.view(nb, NL, H * G, D).to(torch.bfloat16)
    return out


def algorithmic_bytes(resident_rows: int, batch: int, num_layers: int, q_heads: int,
                      head_dim: int = 128) -> int:
    """resident K+V (bf16) plus Q in / O out per step."""
    return resident_rows * 2 * head_dim * 2 + batch * num_layers * q_heads * head_dim * 2 * 2
