"""Brute-force references for tiny codes (independent of both oracle and CUDA path).

These enumerate all 2^n binary vectors, so n must stay <= ~18.  They restate
the textbook definitions the BP decoder is pinned to (SURVEY.md §8(c) "What
pins each part"): exact bit-wise MAP marginals of P(u | L, H u = s) and
syndrome-constrained ML decoding.
"""
from __future__ import annotations

import itertools

import numpy as np


def all_vectors(n: int) -> np.ndarray:
    return np.array(list(itertools.product([0, 1], repeat=n)), dtype=np.uint8)[:, ::-1].copy()


def coset(H: np.ndarray, s: np.ndarray) -> np.ndarray:
    U = all_vectors(H.shape[1])
    ok = np.all((U.astype(np.int64) @ H.T.astype(np.int64)) % 2 == s[None, :], axis=1)
    return U[ok]


def exact_marginal_llr(H: np.ndarray, s: np.ndarray, L: np.ndarray) -> np.ndarray:
    """ln P(u_v=0 | L, Hu=s) - ln P(u_v=1 | ...), with P(u) ∝ prod_v exp(-u_v L_v)."""
    C = coset(H, s).astype(np.float64)
    logw = -(C @ L)
    mx = logw.max()
    w = np.exp(logw - mx)
    out = np.empty(H.shape[1])
    for v in range(H.shape[1]):
        w0 = w[C[:, v] == 0].sum()
        w1 = w[C[:, v] == 1].sum()
        out[v] = np.log(w0) - np.log(w1)
    return out


def ml_decode(H: np.ndarray, s: np.ndarray, L: np.ndarray) -> np.ndarray:
    C = coset(H, s)
    return C[np.argmax(-(C.astype(np.float64) @ L))]


def random_tree_code(rng: np.random.Generator, n_checks: int, max_dc: int = 4):
    """Random cycle-free Tanner graph: checks attached one at a time, each new check
    sharing exactly one variable with the existing tree plus fresh variables."""
    rows = []
    n = 0
    for c in range(n_checks):
        d = int(rng.integers(2, max_dc + 1))
        if c == 0:
            row = list(range(d))
            n = d
        else:
            shared = int(rng.integers(0, n))
            fresh = list(range(n, n + d - 1))
            n += d - 1
            row = [shared] + fresh
        rows.append(sorted(row))
    H = np.zeros((n_checks, n), np.uint8)
    for c, r in enumerate(rows):
        H[c, r] = 1
    return H


def pack_bits(b: np.ndarray) -> np.ndarray:
    """uint8[F][n] 0/1 -> uint32[F][ceil(n/32)], bit i at (i mod 32) of word i/32."""
    b = np.atleast_2d(np.asarray(b, np.uint8))
    F, n = b.shape
    W = (n + 31) // 32
    pad = np.zeros((F, W * 32), np.uint8)
    pad[:, :n] = b
    bits = pad.reshape(F, W, 32).astype(np.uint64)
    return (bits << np.arange(32, dtype=np.uint64)).sum(axis=2).astype(np.uint32)


def unpack_bits(w: np.ndarray, n: int) -> np.ndarray:
    w = np.atleast_2d(np.asarray(w, np.uint32))
    F = w.shape[0]
    bits = (w[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(F, -1)[:, :n].astype(np.uint8)
