"""HeteroCache-B200: the HeteroCache (arXiv 2601.13684) decode hot path, B200-native.

Host mirror of the reference ``heterocache`` API (engine / metrics / budget /
profiling / reporting / trace) over hand-written sm_100a kernels behind a C
ABI (include/hcb200.h, libhcb200.so).  There is no CPU fallback.
"""

__version__ = "0.1.0"
