"""fp32 CPU attention oracle -- TEST INFRASTRUCTURE ONLY (parity unpinned).

The reference package never touches K/V tensors, so
attention outputs have no reference implementation to pin against.  This is a
new fp32 restatement of the score semantics the reference's trace exporter
defines:

* per query head: softmax(q . K^T / sqrt(d)) over the visible span, then
  P . V  (pkg/exporter/src/model.ts:232-270, tools/check_heads.py:85-119);
* per KV head: the recorded attention row is the mean over its G query heads
  of the post-softmax probabilities, added in query-head order then divided by
  G (model.ts:274-291, check_heads.py:119);
* the visible span of a head at decode step t is exactly the CacheView
  resident set (engine.py:98-115): all of [0, L+t) for full heads, and
  dynamic U sinks U recency tail U decode appends for compressed heads.

Inputs are the bf16 tensors the GPU consumed, upcast exactly to fp32; all
arithmetic is fp32 (torch CPU, all host threads).  Only tests/, smoke() and
bench.py's CPU baseline may use it.
"""

from __future__ import annotations

import math

import torch


def unit_attention(q, k, v, positions=None):
    """One KV head: q [G, d], k/v [n, d] (any float dtype), positions: the
    resident row ids (None = all rows).  Returns (o [G, d] fp32,
    probs [G, n_res] fp32, positions used)."""
    q = q.float()
    k = k.float()
    v = v.float()
    if positions is not None:
        pos = torch.as_tensor(positions, dtype=torch.long)
        k = k.index_select(0, pos)
        v = v.index_select(0, pos)
    d = q.shape[-1]
    s = (q @ k.T) * (1.0 / math.sqrt(d))
    s = s - s.max(dim=-1, keepdim=True).values
    e = torch.exp(s)
    p = e * (1.0 / e.sum(dim=-1, keepdim=True))
    return p @ v, p


def gqa_mean_row(probs):
    """Mean over query heads, added in head order then / G (model.ts:283-289)."""
    acc = torch.zeros_like(probs[0])
    for j in range(probs.shape[0]):
        acc = acc + probs[j]
    return acc / probs.shape[0]


def decode_step_reference(q, kv_rows, resident):
    """Whole-step oracle.

    q: dict unit -> [G, d]; kv_rows: dict unit -> (K [n, d], V [n, d]) holding
    the head's full position-indexed KV (row p = position p); resident: dict
    unit -> sorted position list.  Returns dict unit -> (o [G, d], row) where
    row is the GQA-mean probability row over the resident positions.
    """
    out = {}
    for u, qu in q.items():
        k, v = kv_rows[u]
        o, p = unit_attention(qu, k, v, resident[u])
        out[u] = (o, gqa_mean_row(p))
    return out
