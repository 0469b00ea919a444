"""Host twin of the bench's synthetic generator -- TEST / BASELINE INFRASTRUCTURE.

`HostNormal` is the `normal` hook of paper_2601_13684_b200.workload.SyntheticKV
for the CPU arms of bench.py (reference arm, cpu_baseline leg) and for tests:
oracle/synth.c reproduces csrc/synth.cu bit for bit, so a CPU-side
SyntheticKV(..., normal=HostNormal(), seqs=[...]) yields exactly the K/V/Q
slices the GPU arm decodes.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        from . import build_oracle

        path = build_oracle.LIB
        if not path.exists():
            build_oracle.build()
        lib = C.CDLL(str(path))
        lib.oracle_synth_normal.restype = None
        lib.oracle_synth_normal.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int64]
        _LIB = lib
    return _LIB


class HostNormal:
    """N(key, offset + i) as a CPU float32 torch tensor (OpenMP, all cores)."""

    device = "cpu"

    def __call__(self, shape, key: int, offset: int = 0):
        import torch

        out = torch.empty(shape, dtype=torch.float32)
        _lib().oracle_synth_normal(out.data_ptr(), out.numel(), key & ((1 << 64) - 1), offset)
        return out
