"""B200-native importance-sampled mini-batch SGD for CP decomposition (arXiv 2103.04081).

The hot path (sampling, fiber gather, sampled Khatri-Rao rows, reweighted gradient, fixed /
adaptive update, table refresh) runs in hand-written sm_100a kernels behind the C ABI of
``include/cpsgd.h`` (``libcpsgd.so``); this package is a thin ctypes binding plus host-side
plumbing (slab sharding helpers).  There is no CPU fallback.
"""
from .cpsgd import CPSGD, CPError, load_library, LIB_PATH, SAMPLERS, RULES  # noqa: F401

__all__ = ["CPSGD", "CPError", "load_library", "LIB_PATH", "SAMPLERS", "RULES"]
