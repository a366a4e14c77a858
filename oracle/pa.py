"""Privacy-amplification oracle (numpy, bit by bit).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module; the product path never does.

PAPER.md:92 (Step 6): Alice and Bob "apply a 2-universal hashing function on
their reconciled string to obtain two identical and shorter secret key
strings".  The paper names no family; reading R-8 fixes the Toeplitz
family: a seed t of n_in + n_out - 1 bits defines
T in {0,1}^{n_out x n_in},

    T[i][j] = t[i - j + n_in - 1],      y = T x  over GF(2),

i.e. y_i = XOR_j t[i - j + n_in - 1] AND x_j, evaluated here row by row.
Pinned in tests/test_oracle_pins.py (numpy convolution window, unit and
all-ones seeds, linearity, 2-universality statistics).
"""
from __future__ import annotations

import numpy as np


def toeplitz_row(t: np.ndarray, n_in: int, i: int) -> np.ndarray:
    """Row i of T: T[i][j] = t[i - j + n_in - 1] for j = 0..n_in-1."""
    idx = i + n_in - 1 - np.arange(n_in)
    return np.asarray(t, dtype=np.uint8)[idx]


def toeplitz_hash(t: np.ndarray, x: np.ndarray, n_out: int, rows=None) -> np.ndarray:
    """y = T x over GF(2) for 0/1 arrays t (n_in + n_out - 1) and x (n_in); `rows` selects
    a subset of output indices (sampled parity at large sizes)."""
    x = np.asarray(x, dtype=np.uint8)
    n_in = x.size
    if np.asarray(t).size != n_in + n_out - 1:
        raise ValueError("seed must have n_in + n_out - 1 bits")
    rows = range(n_out) if rows is None else rows
    return np.array([int(np.bitwise_xor.reduce(toeplitz_row(t, n_in, i) & x)) if n_in else 0 for i in rows],
                    dtype=np.uint8)


def pack_bits(b: np.ndarray) -> np.ndarray:
    """0/1 array -> uint32 words, bit i at bit (i % 32) of word i // 32."""
    b = np.asarray(b, dtype=np.uint8).ravel()
    pad = np.zeros((-b.size) % 32, np.uint8)
    return np.packbits(np.concatenate([b, pad]), bitorder="little").view("<u4").copy()


def unpack_bits(w: np.ndarray, nbits: int) -> np.ndarray:
    return np.unpackbits(np.asarray(w, dtype="<u4").view(np.uint8), bitorder="little")[:nbits]
