"""Quantiser parameter table (input, not arithmetic of the method).

Reading A-3 of PAPER.md:132 ("a constant quantisation size
of the real line across 2^5 bins centered on zero"): bin edges at integer
multiples of the step delta, symmetric about zero, outer bins unbounded:

    e_k = fp32((k - 2^(m-1)) * delta),   k = 1 .. 2^m - 1.

The fp32 table is computed once here (double -> float) and handed to both the
CUDA path and the oracle, so that the quantiser comparison y >= e_k is
bit-exact on both sides.
"""
from __future__ import annotations

import numpy as np


def edge_table(m: int, delta: float) -> np.ndarray:
    if not (1 <= m <= 8):
        raise ValueError("m must be in [1, 8]")
    if m > 1 and not delta > 0:
        raise ValueError("delta must be > 0")
    k = np.arange(1, 2 ** m, dtype=np.float64)
    return ((k - 2 ** (m - 1)) * float(delta)).astype(np.float32)
