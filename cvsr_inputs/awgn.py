"""Seeded synthetic inputs (input generator shared by the CUDA path and the oracle).

Quadratures follow PAPER.md:361-365 (Section V, "we can generate these
quadrature values"): Alice's x are Gaussian and Bob's y = x + n with
n ~ N(0, sigma_n^2).  Reading A-5: SNR = gamma, i.e.
x ~ N(0, 1) and n ~ N(0, 1/gamma), so sigma_n = gamma^-1/2 in units of sigma_x.

Seeding: every frame f draws from its own Philox stream keyed (seed, f), so a
frame's data is independent of batch size, frame order and GPU count
(SURVEY.md §8(d) "Seeds").  Values are produced in float64 and rounded once
to float32, the ABI's input type.
"""
from __future__ import annotations

import numpy as np

DATA_SEED = 210808418


def _gen(seed: int, frame: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, frame]))


def quadratures(frames: int, n: int, gamma: float, seed: int = DATA_SEED,
                first_frame: int = 0):
    """(x, y) float32[frames][n] per PAPER.md:361-365 with reading A-5."""
    sigma_n = 1.0 / np.sqrt(gamma)
    x = np.empty((frames, n), np.float32)
    y = np.empty((frames, n), np.float32)
    for i in range(frames):
        g = _gen(seed, first_frame + i)
        xd = g.standard_normal(n)
        yd = xd + sigma_n * g.standard_normal(n)
        x[i] = xd.astype(np.float32)
        y[i] = yd.astype(np.float32)
    return x, y


def biawgn(frames: int, n: int, sigma: float, seed: int = DATA_SEED, first_frame: int = 0):
    """BI-AWGN decoder-only inputs (config C1, reading A-16): u ~ Bernoulli(1/2),
    y = 1 - 2u + sigma*noise.  Returns (u uint8[frames][n], y float32[frames][n])."""
    u = np.empty((frames, n), np.uint8)
    y = np.empty((frames, n), np.float32)
    for i in range(frames):
        g = _gen(seed, first_frame + i)
        ui = g.integers(0, 2, n, dtype=np.uint8)
        u[i] = ui
        y[i] = ((1.0 - 2.0 * ui) + sigma * g.standard_normal(n)).astype(np.float32)
    return u, y


def biawgn_sigma(rate: float, ebn0_db: float) -> float:
    """sigma for BPSK at E_b/N_0 (reading A-16): sigma^2 = 1 / (2 R 10^(EbN0/10))."""
    return float(np.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0))))


def torch_quadratures(frames: int, n: int, gamma: float, device, seed: int = DATA_SEED,
                      first_frame: int = 0, chunk: int = 64):
    """Device-side generator for benchmark-size batches (torch Philox per frame chunk).

    Frames are generated in GLOBAL chunks of `chunk` frames, chunk c seeded by
    (seed, c), so frame f's data does not depend on how frames are sharded
    across ranks.  Different bits from :func:`quadratures` (another generator)
    but the same distribution; both implementations consume whatever arrays
    are produced, so parity is unaffected.
    """
    import torch
    sigma_n = float(1.0 / np.sqrt(gamma))
    x = torch.empty((frames, n), dtype=torch.float32, device=device)
    y = torch.empty((frames, n), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    last = first_frame + frames
    for cid in range(first_frame // chunk, (last + chunk - 1) // chunk):
        g.manual_seed((seed * 1000003 + cid) & 0x7FFFFFFFFFFFFFFF)
        xs = torch.randn((chunk, n), generator=g, device=device, dtype=torch.float32)
        ns = torch.randn((chunk, n), generator=g, device=device, dtype=torch.float32)
        lo, hi = max(first_frame, cid * chunk), min(last, (cid + 1) * chunk)
        a, b = lo - cid * chunk, hi - cid * chunk
        x[lo - first_frame:hi - first_frame] = xs[a:b]
        y[lo - first_frame:hi - first_frame] = xs[a:b] + sigma_n * ns[a:b]
    return x, y
