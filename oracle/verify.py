"""Verification-hash oracle (plain Python integers).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module; the product path never does.

PAPER.md:90 (Step 5, last paragraph): "Alice and Bob obtain two hashed strings
by applying the same hash function to their reconciled strings and exchange the
hash results to check whether SR is successful."  The paper names no hash
function; reading R-6 fixes it to the polynomial (Carter-Wegman) hash
over GF(p), p = 2^61 - 1, applied per frame (sub-block):

    h(w; key) = sum_{i=0}^{W-1} w_i * key^(i+1)  mod p,

w_i = the i-th little-endian 32-bit word of the frame's label bytes, zero-padded
to W = ceil(n/4) words.  Two different strings collide for at most W of the
p - 1 keys (a nonzero polynomial of degree <= W has <= W roots).  The check of
PAPER.md:90 uses 3 independent keys (cvsr_verify): a wrong frame passes with
probability <= (W/(p-1))^3 <= 2^-122 up to n = 5e6.  (PAPER.md:354 quotes a
hashing parameter eps_h = 4.7e-13 for the alternate key-rate equation of
[pirandola2021limits]; the adopted equation charges reconciliation failure to
eps_EC.)

Pinned in tests/test_oracle_pins.py (key = 1 is the word checksum, key = 2^32
is 2^32 * int.from_bytes(label, 'little') mod p, zero string, padding).
"""
from __future__ import annotations

import numpy as np

P61 = (1 << 61) - 1


def frame_words(label_row: np.ndarray) -> list:
    """The W = ceil(n/4) little-endian 32-bit words of one frame's label bytes."""
    b = bytes(np.asarray(label_row, dtype=np.uint8).tobytes())
    b += b"\0" * ((-len(b)) % 4)
    return [b[4 * i] | (b[4 * i + 1] << 8) | (b[4 * i + 2] << 16) | (b[4 * i + 3] << 24)
            for i in range(len(b) // 4)]


def frame_hash(label: np.ndarray, key: int) -> np.ndarray:
    """h per frame of label uint8[F][n] (definition above, evaluated term by term)."""
    if not (1 <= key <= P61 - 2):
        raise ValueError("key must be in [1, 2^61 - 2]")
    label = np.atleast_2d(np.asarray(label, dtype=np.uint8))
    out = np.zeros(label.shape[0], dtype=np.uint64)
    for f in range(label.shape[0]):
        h = 0
        kp = 1
        for w in frame_words(label[f]):
            kp = (kp * key) % P61          # key^(i+1)
            h = (h + w * kp) % P61
        out[f] = h
    return out
