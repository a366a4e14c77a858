"""B200-native (sm_100a) sliced reconciliation hot path for CV-QKD (arXiv 2108.08418).

The product is libcvsr.so (C ABI in include/cvsr.h); ``cvsr`` is its thin
ctypes binding and ``pipeline`` composes the ABI calls into one
Bob + Alice step for benchmarks.  There is no CPU fallback.
"""
from ._build import LIB, build  # noqa: F401


def load():
    """Import the binding (raises if libcvsr.so is missing)."""
    from . import cvsr
    return cvsr
