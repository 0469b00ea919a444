"""ctypes binding of the C ABI in include/hcb200.h (libhcb200.so).

There is no fallback: if the library is missing or no CUDA device is
present, every compute entry point raises.  PyTorch is used only for device
memory and streams; all compute goes through the kernels behind this ABI.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libhcb200.so"

HC_OK, HC_EINVAL, HC_EINFEASIBLE, HC_ECUDA, HC_ENOMEM, HC_ESTATE = range(6)
PAD_INDEX = 0xFFFFFFFF

u32p = C.POINTER(C.c_uint32)


class HCError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hcb200 error {code}: {msg}")
        self.code = code


class TopkJob(C.Structure):
    _fields_ = [
        ("scores", C.c_void_p), ("idx", C.c_void_p), ("n", C.c_uint32), ("k", C.c_uint32),
        ("out_idx", C.c_void_p), ("out_count", C.c_void_p), ("base_bitmap", C.c_void_p),
        ("overlap_out", C.c_void_p),
    ]


class EngineDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "batch", "num_layers", "kv_heads", "group", "head_dim", "prefill_len", "max_decode",
        "sink_count", "recency_window", "l_base_int", "chunk", "monitor", "host_pool",
        "obs_window", "score_material", "device_decisions", "window", "update_delay_steps",
        "eval_every_step", "bytes_per_kv_entry", "pad_")] + [
        ("transfer_bandwidth", C.c_int64), ("tau_drift", C.c_double)]


class FireRecord(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "trigger_step", "pivot_unit", "completion_step", "n_satellites")] + [
        ("transfer_bytes", C.c_int64), ("cumulative_bytes", C.c_int64),
        ("first_satellite", C.c_int32), ("fetched_offset", C.c_int32),
        ("fetched_counts", C.c_int32 * 8)]


class RecallHead(C.Structure):
    _fields_ = [("idx", C.c_void_p), ("scores", C.c_void_p), ("dynamic", C.c_void_p)]


_lib = None


def _declare(lib):
    vp, i32, u32 = C.c_void_p, C.c_int, C.c_uint32
    sig = {
        "hc_version": (C.c_char_p, []),
        "hc_last_error": (C.c_char_p, []),
        "hc_launch_count": (C.c_ulonglong, []),
        "hc_topk_batched": (i32, [vp, i32, u32, vp]),
        "hc_select_topk": (i32, [vp, vp, u32, u32, vp, vp, vp]),
        "hc_bitmap_from_indices": (i32, [vp, u32, vp, vp, u32, vp]),
        "hc_monitor_rows": (i32, [vp, C.c_int64, i32, u32, u32, vp, i32, vp, vp, vp]),
        "hc_obs_scores": (i32, [vp, vp, i32, i32, i32, i32, i32, vp, C.c_int64, vp]),
        "hc_gram_from_sets": (i32, [vp, vp, i32, i32, i32, i32, vp, vp]),
        "hc_trace_recall": (i32, [vp, i32, u32, C.c_uint64, u32, u32, u32, u32, vp, vp]),
        "hc_engine_create": (i32, [vp, vp, vp, vp, vp]),
        "hc_engine_create_sharded": (i32, [vp, vp, vp, vp, vp, vp]),
        "hc_engine_destroy": (i32, [vp]),
        "hc_engine_info": (i32, [vp, vp]),
        "hc_engine_prefill_layer": (i32, [vp, i32, vp, vp, vp, vp]),
        "hc_engine_decode_step": (i32, [vp, i32, vp, vp, vp, vp, vp]),
        "hc_engine_decode_begin": (i32, [vp, i32, vp, vp, vp, vp, i32, vp]),
        "hc_engine_decode_end": (i32, [vp, i32, vp]),
        "hc_engine_decode_step_host": (i32, [vp, i32, vp, vp, vp, vp, vp]),
        "hc_engine_join": (i32, [vp, vp]),
        "hc_pooled_topk": (i32, [vp, u32, u32, u32, vp, vp]),
        "hc_engine_enable_measure": (i32, [vp, i32]),
        "hc_engine_measure": (i32, [vp, i32, vp, vp, vp]),
        "hc_engine_measure_records": (i32, [vp, i32, vp, vp, i32, vp]),
        "hc_engine_overlaps": (i32, [vp, i32, i32, vp, vp]),
        "hc_engine_fire": (i32, [vp, i32, i32, i32, vp, vp]),
        "hc_engine_land": (i32, [vp, i32, vp]),
        "hc_engine_wait_fetched": (i32, [vp]),
        "hc_engine_poll_decisions": (i32, [vp, i32, vp, vp, i32, vp, vp, C.c_int64]),
        "hc_engine_devdec_satellites": (i32, [vp, vp, i32, vp]),
        "hc_engine_fire_batch": (i32, [vp, i32, vp, i32, vp, vp, vp, vp]),
        "hc_engine_land_batch": (i32, [vp, i32, vp, vp]),
        "hc_engine_read_indices": (i32, [vp, i32, i32, vp, i32, vp, vp]),
        "hc_engine_pivot_row": (i32, [vp, i32, i32, vp, vp]),
        "hc_engine_resident_rows": (i32, [vp, i32, vp, vp]),
        "hc_engine_set_prefill_dump": (i32, [vp, vp]),
        "hc_engine_active_tiles": (i32, [vp, i32, vp]),
        "hc_engine_timing": (i32, [vp, i32, vp, vp]),
        "hc_engine_retrieval_stats": (i32, [vp, vp]),
        "hc_engine_gaps": (i32, [vp, vp, i32, vp]),
        "hc_engine_prefill_stats": (i32, [vp, vp]),
        "hc_synth_normal": (i32, [vp, C.c_int64, C.c_uint64, C.c_int64, vp]),
        "hc_read_probe": (i32, [vp, C.c_int64, vp, i32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return sig


EXPORTED = None


def load():
    """Load (never build) the shared library; raises if it is absent."""
    global _lib, EXPORTED
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("HCB200_LIB", LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2601_13684_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(path))
    EXPORTED = sorted(_declare(lib))
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != HC_OK:
        msg = load().hc_last_error().decode(errors="replace")
        raise HCError(rc, msg)


def ptr(t) -> int:
    """Device (or host) address of a torch tensor, or 0 for None."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    """cudaStream_t of `stream`, or of torch's current stream (raw query: the public
    torch.cuda.current_stream() costs ~15 us per call, a quarter of a small step's host time)."""
    if stream is not None:
        return int(stream.cuda_stream)
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(torch._C._cuda_getDevice()))
    return int(torch.cuda.current_stream().cuda_stream)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise HCError(HC_ECUDA, "no CUDA device: the HeteroCache-B200 path has no CPU fallback")
    load()
