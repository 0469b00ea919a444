"""Thin Python wrappers over the C ABI (device memory via torch, compute via CUDA).

Every function here launches kernels from libhcb200.so; nothing computes on
the CPU.  They exist for the host mirror (engine.py, profiling.py) and for
parity tests.
"""

from __future__ import annotations

import numpy as np

from . import _lib

TOPK_JOB_DTYPE = np.dtype({
    "names": ["scores", "idx", "n", "k", "out_idx", "out_count", "base_bitmap", "overlap_out"],
    "formats": ["<u8", "<u8", "<u4", "<u4", "<u8", "<u8", "<u8", "<u8"],
    "offsets": [0, 8, 16, 20, 24, 32, 40, 48],
    "itemsize": 56,
})
RECALL_HEAD_DTYPE = np.dtype({
    "names": ["idx", "scores", "dynamic"],
    "formats": ["<u8", "<u8", "<u8"],
    "offsets": [0, 8, 16],
    "itemsize": 24,
})


def _torch():
    import torch

    return torch


def to_device_struct(arr: np.ndarray, device="cuda"):
    """Upload a numpy structured array as raw bytes; returns a uint8 tensor."""
    torch = _torch()
    raw = np.frombuffer(arr.tobytes(), dtype=np.uint8)
    return torch.from_numpy(raw.copy()).to(device, non_blocking=False)


def launch_topk(jobs: np.ndarray, n_add: int = 0, stream=None, jobs_dev=None):
    """Launch K1 over a TOPK_JOB_DTYPE array (or its uploaded copy)."""
    lib = _lib.load()
    if len(jobs) == 0:
        return None
    if jobs_dev is None:
        jobs_dev = to_device_struct(jobs)
    _lib.check(lib.hc_topk_batched(_lib.ptr(jobs_dev), len(jobs), n_add,
                                   _lib.stream_handle(stream)))
    return jobs_dev


def topk_rows(idx, scores, k, base_bitmaps=None):
    """Top-k of every row of (idx, scores) (idx None = dense rows).

    k: int or per-row sequence.  Returns (selected [R, kmax] uint32 with the
    selected token indices in candidate order, counts [R] uint32) as numpy;
    with base_bitmaps ([R, words] uint32 or None) also returns overlaps [R].
    """
    torch = _torch()
    _lib.require_cuda()
    sc = torch.from_numpy(np.array(scores, dtype=np.float32, order="C")).cuda()
    R, K = sc.shape
    ix = None
    if idx is not None:
        ix = torch.from_numpy(np.array(idx, dtype=np.uint32, order="C").view(np.int32)).cuda()
    ks = np.broadcast_to(np.asarray(k, dtype=np.int64), (R,))
    kmax = int(max(1, ks.max())) if R else 1
    out = torch.zeros((R, kmax), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(R, dtype=torch.int32, device="cuda")
    ovl = torch.zeros(R, dtype=torch.int32, device="cuda")
    bm = None
    if base_bitmaps is not None:
        bm = torch.from_numpy(np.array(base_bitmaps, dtype=np.uint32, order="C")
                              .view(np.int32)).cuda()
    jobs = np.zeros(R, dtype=TOPK_JOB_DTYPE)
    row_bytes = K * 4
    jobs["scores"] = _lib.ptr(sc) + np.arange(R, dtype=np.uint64) * row_bytes
    if ix is not None:
        jobs["idx"] = _lib.ptr(ix) + np.arange(R, dtype=np.uint64) * row_bytes
    jobs["n"] = K
    jobs["k"] = ks
    jobs["out_idx"] = _lib.ptr(out) + np.arange(R, dtype=np.uint64) * (kmax * 4)
    jobs["out_count"] = _lib.ptr(cnt) + np.arange(R, dtype=np.uint64) * 4
    if bm is not None:
        jobs["base_bitmap"] = _lib.ptr(bm) + np.arange(R, dtype=np.uint64) * (bm.shape[1] * 4)
        jobs["overlap_out"] = _lib.ptr(ovl) + np.arange(R, dtype=np.uint64) * 4
    dev = launch_topk(jobs)
    torch.cuda.synchronize()
    del dev
    sel = out.cpu().numpy().view(np.uint32)
    counts = cnt.cpu().numpy().view(np.uint32)
    if base_bitmaps is not None:
        return sel, counts, ovl.cpu().numpy().view(np.uint32)
    return sel, counts


def top_k_indices(scores, k: int, pool_kernel: int = 0) -> frozenset:
    """Drop-in for heterocache.metrics.top_k_indices (metrics.py:48-71), on the GPU.

    Dense 1-D arrays and (index, score) pair sequences are supported.  Dense
    rows with pool_kernel > 0 take the pooled path (hc_pooled_topk: float64
    moving sums in numpy's order, then the (pooled, raw, index) order of
    metrics.py:26-39); the engine itself never pools (engine.py:229-230).
    """
    if k < 0:
        raise ValueError(f"k must be nonnegative, got {k}")
    if k == 0:
        return frozenset()
    if pool_kernel:
        return _pooled_top_k(scores, k, pool_kernel)
    if isinstance(scores, np.ndarray):
        row = np.asarray(scores, dtype=np.float64)
        if row.ndim != 1:
            raise ValueError(f"dense scores must be 1-D, got shape {row.shape}")
        f32 = row.astype(np.float32)
        if not np.array_equal(f32.astype(np.float64), row):
            raise ValueError("dense scores must be exactly representable in float32")
        sel, cnt = topk_rows(None, f32[None, :], k)
        return frozenset(int(x) for x in sel[0, :cnt[0]])
    seq = list(scores)
    if not seq:
        return frozenset()
    if isinstance(seq[0], (tuple, list)) and len(seq[0]) == 2:
        idx = np.array([int(i) for i, _ in seq], dtype=np.uint32)
        sc = np.array([float(s) for _, s in seq], dtype=np.float32)
        sel, cnt = topk_rows(idx[None, :], sc[None, :], k)
        return frozenset(int(x) for x in sel[0, :cnt[0]])
    return top_k_indices(np.asarray(seq, dtype=np.float64), k)


def _pooled_top_k(scores, k: int, pool_kernel: int) -> frozenset:
    w = np.asarray(scores, dtype=np.float64)
    if w.ndim != 1:
        raise ValueError(f"dense scores must be 1-D, got shape {w.shape}")
    if pool_kernel < 1 or pool_kernel % 2 == 0:
        raise ValueError(f"pool kernel must be odd and positive, got {pool_kernel}")
    if pool_kernel > w.size:  # np.convolve 'same' returns max(n, kernel) values: lexsort refuses
        raise ValueError("all keys need to be the same shape")
    torch = _torch()
    _lib.require_cuda()
    d = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    out = torch.empty(min(k, w.size), dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().hc_pooled_topk(_lib.ptr(d), w.size, pool_kernel, k, _lib.ptr(out),
                                          _lib.stream_handle()))
    return frozenset(int(x) for x in out.cpu().numpy())


def monitor_rows(rows, k: int, base_bitmaps):
    """Drift-monitor K1+K2 over dense rows: (thresholds [R] uint64, overlaps [R])."""
    torch = _torch()
    _lib.require_cuda()
    R, n = rows.shape
    stride = (n + 3) // 4 * 4
    dev = torch.zeros((R, stride), dtype=torch.float32, device="cuda")
    dev[:, :n] = torch.as_tensor(np.asarray(rows, dtype=np.float32))
    words = base_bitmaps.shape[1]
    bm = torch.as_tensor(np.ascontiguousarray(base_bitmaps, dtype=np.uint32).view(np.int32)).cuda()
    thr = torch.zeros(R, dtype=torch.int64, device="cuda")
    ovl = torch.zeros(R, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().hc_monitor_rows(_lib.ptr(dev), stride, R, n, k, _lib.ptr(bm), words,
                                           _lib.ptr(thr), _lib.ptr(ovl), _lib.stream_handle()))
    return thr.cpu().numpy().view(np.uint64), ovl.cpu().numpy()
