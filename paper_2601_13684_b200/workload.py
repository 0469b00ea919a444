"""Synthetic decode workloads: model shapes, head roles,
budgets and seeded bf16 K/V/Q with planted hot sets and topic shifts.

Everything is generated on the device (torch RNG) so 128K-224K contexts never
touch host memory.  Roles per layer follow the survey's synthetic mix:
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


class SyntheticKV:
    """Seeded K/V/Q with planted per-cluster hot sets and topic shifts.

    For each (sequence b, layer l) the cluster (pivot + satellites) shares two
    topic directions u0/u1 with hot position sets H0/H1; anchors own a fixed
    topic; the volatile head attends diffusely.  Keys at hot positions get
    +alpha*u, queries are beta*u(t) + N(0, I) with the cluster topic switching
    from u0 to u1 at the shift step, so the pivot's top set moves and the drift
    monitor fires (engine.py:313-321).
    """

    def __init__(self, model: ModelShape, *, batch: int, prefill_len: int, num_layers: int,
                 hot: int, seed: int, alpha: float = 9.0, beta: float = 9.0, device="cuda"):
        import torch

        self.torch = torch
        self.m, self.B, self.L, self.NL = model, batch, prefill_len, num_layers
        self.D, self.H, self.G = model.head_dim, model.kv_heads, model.group
        self.hot, self.seed, self.alpha, self.beta, self.dev = hot, seed, alpha, beta, device
        self.roles = model.layer_roles()
        g = torch.Generator(device="cpu").manual_seed(seed)
        # per (b, l): topic directions [B, NL, 3 topics, D] (0/1: cluster, 2: anchor)
        u = torch.randn(batch, num_layers, 3, self.D, generator=g)
        self.u = (u / u.norm(dim=-1, keepdim=True)).to(device)
        hot = min(hot, prefill_len // 4)
        self.hot_sets = torch.stack([
            torch.stack([torch.randperm(prefill_len, generator=g)[:3 * hot].view(3, hot)
                         for _ in range(num_layers)]) for _ in range(batch)]).to(device)

    def _head_topic(self, h: int) -> int:
        r = self.roles[h]
        return {"pivot": 0, "satellite": 0, "anchor": 2, "volatile": -1}[r]

    def layer_kv(self, layer: int, window: int = 1):
        """K, V [B, H, L, D] bf16 and the prefill observation queries for one layer:
        q_last [B, H*G, D] (window 1) or [B, window, H*G, D] (last `window` tokens)."""
        torch = self.torch
        g = torch.Generator(device=self.dev).manual_seed(self.seed * 1000 + layer)
        B, H, L, D = self.B, self.H, self.L, self.D
        k = torch.randn(B, H, L, D, device=self.dev, generator=g, dtype=torch.float32)
        v = torch.randn(B, H, L, D, device=self.dev, generator=g, dtype=torch.float32)
        for h in range(H):
            tp = self._head_topic(h)
            if tp < 0:
                continue
            for topic in ((0, 1) if tp == 0 else (2,)):
                idx = self.hot_sets[:, layer, topic]                      # [B, hot]
                add = self.alpha * self.u[:, layer, topic]               # [B, D]
                k[:, h].scatter_add_(1, idx[:, :, None].expand(-1, -1, D),
                                     add[:, None, :].expand(-1, idx.shape[1], -1).contiguous())
        if window == 1:
            q = self.queries(layer, 0)
        else:
            q = torch.stack([self.queries(layer, -1 - i) for i in range(window)][::-1], dim=1)
        return k.to(torch.bfloat16).contiguous(), v.to(torch.bfloat16).contiguous(), q.contiguous()

    def queries(self, layer: int, step: int, shift_step=None):
        """[B, H*G, D] bf16 queries of one layer at a decode step.  shift_step: the
        step of the planted topic shift, or a sequence of shift steps (the cluster
        topic toggles at each)."""
        torch = self.torch
        g = torch.Generator(device=self.dev).manual_seed((self.seed * 7919 + layer) * 100003 + step)
        B, H, G, D = self.B, self.H, self.G, self.D
        q = torch.randn(B, H, G, D, device=self.dev, generator=g)
        for h in range(H):
            tp = self._head_topic(h)
            if tp < 0:
                continue
            if tp == 0 and shift_step is not None:
                shifts = shift_step if isinstance(shift_step, (list, tuple)) else (shift_step,)
                tp = sum(step >= x for x in shifts) % 2
            q[:, h] += self.beta * self.u[:, layer, tp][:, None, :]
        return q.view(B, H * G, D).to(torch.bfloat16).contiguous()

    def step_inputs(self, step: int, shift_step: int | None):
        """q [B, NL, H*G, D], k_new/v_new [B, NL, H, D] (bf16, device)."""
        torch = self.torch
        q = torch.stack([self.queries(l, step, shift_step) for l in range(self.NL)], dim=1)
        g = torch.Generator(device=self.dev).manual_seed(self.seed * 31 + step)
        kn = torch.randn(self.B, self.NL, self.H, self.D, device=self.dev, generator=g)
        vn = torch.randn(self.B, self.NL, self.H, self.D, device=self.dev, generator=g)
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
    """Queries for decode steps 1..steps: [steps + 1, B, NL, H*G, D] bf16 (device).

    Cluster heads (pivot, satellites) of (b, l) follow topic u0 or u1, toggling at
    each of that cluster's shift steps; noise cycles through n_noise draws."""
    torch = gen.torch
    B, NL, H, G, D = gen.B, gen.NL, gen.H, gen.G, gen.D
    noise = []
    for i in range(n_noise):
        g = torch.Generator(device=gen.dev).manual_seed(gen.seed * 131 + i)
        noise.append(torch.randn(B, NL, H, G, D, device=gen.dev, generator=g))
    cluster = torch.tensor([gen._head_topic(h) == 0 for h in range(H)], device=gen.dev)
    anchor = torch.tensor([gen._head_topic(h) == 2 for h in range(H)], device=gen.dev)
    u = gen.u  # [B, NL, 3, D]
    out = torch.empty(steps + 1, B, NL, H * G, D, device=gen.dev, dtype=torch.bfloat16)
    topic = torch.zeros(steps + 1, B, NL, dtype=torch.long, device=gen.dev)
    for (b, l), xs in shifts.items():
        for x in xs:
            if 0 <= x <= steps:
                topic[x:, b, l] ^= 1
    for t in range(steps + 1):
        ut = torch.gather(u, 2, topic[t][:, :, None, None].expand(B, NL, 1, D))[:, :, 0]  # [B,NL,D]
        q = noise[t % n_noise].clone()
        q += gen.beta * (cluster[None, None, :, None, None] * ut[:, :, None, None, :])
        q += gen.beta * (anchor[None, None, :, None, None] * u[:, :, 2][:, :, None, None, :])
        out[t] = q.view(B, NL, H * G, D).to(torch.bfloat16)
    return out


def algorithmic_bytes(resident_rows: int, batch: int, num_layers: int, q_heads: int,
                      head_dim: int = 128) -> int:
    """resident K+V (bf16) plus Q in / O out per step."""
    return resident_rows * 2 * head_dim * 2 + batch * num_layers * q_heads * head_dim * 2 * 2
