"""Host-side analytic formulas of the paper in fp64 (oracle side).  TEST INFRASTRUCTURE ONLY.

Each function restates one PAPER.md equation (cited by its LaTeX label).
Quantised entropies use numerical integration over Alice's x (reading A-5:
x ~ N(0,1), y = x + n, n ~ N(0, 1/gamma)).
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
from scipy import integrate, optimize, special, stats


def snr(V_A: float, T: float, xi_ch: float, xi_d: float) -> float:
    """eq: SNR: gamma = (V_A T / 2) / (1 + xi/2), xi = xi_ch + xi_d."""
    return 0.5 * V_A * T / (1.0 + 0.5 * (xi_ch + xi_d))


def i_ab(gamma: float) -> float:
    """I_AB = C(gamma) = 1/2 log2(1 + gamma) (SPEC.md mutual_information)."""
    return 0.5 * math.log2(1.0 + gamma)


def q_inv(eps: float) -> float:
    """Inverse Q-function (PAPER.md:146-149 defines Q)."""
    return float(stats.norm.isf(eps))


def dispersion(gamma: float, eps_ec: float) -> float:
    """A = (gamma/2) (gamma+2)/(gamma+1)^2 (log eps_EC)^2, natural log."""
    return gamma / 2.0 * (gamma + 2.0) / (gamma + 1.0) ** 2 * math.log(eps_ec) ** 2


def c_finite(gamma: float, n_r: float, eps_ec: float) -> float:
    """eq:R_Finite; log2 in the 1/2 log N_R term (SURVEY App. A reading)."""
    A = dispersion(gamma, eps_ec)
    return i_ab(gamma) - (math.sqrt(n_r * A) * q_inv(eps_ec) + 0.5 * math.log2(n_r)) / n_r


def beta_finite(gamma: float, n_r: float, eps_ec: float) -> float:
    """eq: BetaFinite."""
    return c_finite(gamma, n_r, eps_ec) / i_ab(gamma)


def beta(pi_my: float, m: int, rates: Sequence[float], gamma: float) -> float:
    """equation: beta: (Pi(M(Y)) - m + sum R_j) / I_AB."""
    return (pi_my - m + float(np.sum(rates))) / i_ab(gamma)


def beta2(pi_my: float, m: int, rates: Sequence[float], gamma: float) -> float:
    """equation: beta2: (Pi(M(Y)) - R_s)/I_AB, R_s = sum(1 - R_j)."""
    r_s = float(np.sum([1.0 - r for r in rates]))
    assert len(rates) == m
    return (pi_my - r_s) / i_ab(gamma)


def ops_per_iteration(G: int) -> int:
    """eq: EP: E_j = 7 G, with G = nonzeros of the built H (reading A-20)."""
    return 7 * int(G)


# ---------------------------------------------------------------- quantised entropies

def _edges(m: int, delta: float) -> np.ndarray:
    # fp64 edges at integer multiples of delta (reading A-3); outer bins unbounded
    k = np.arange(1, 2 ** m)
    return (k - 2 ** (m - 1)) * delta


def _bin_probs_given_x(x: np.ndarray, edges: np.ndarray, sigma_n: float) -> np.ndarray:
    """P(bin b | x) for every x (rows) and bin b (cols): Phi differences."""
    z = (edges[None, :] - x[:, None]) / sigma_n
    cdf = special.ndtr(z)
    cdf = np.concatenate([np.zeros((len(x), 1)), cdf, np.ones((len(x), 1))], axis=1)
    return np.clip(np.diff(cdf, axis=1), 0.0, 1.0)


def _xgrid(npts: int = 4001, lim: float = 9.0):
    x = np.linspace(-lim, lim, npts)
    w = stats.norm.pdf(x) * (x[1] - x[0])
    return x, w / w.sum()


def _H(p: np.ndarray, axis=-1) -> np.ndarray:
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.where(p > 0, -p * np.log2(p), 0.0)
    return t.sum(axis=axis)


def entropies(gamma: float, m: int, delta: float, npts: int = 4001):
    """(Pi(M(Y)), Pi(M(Y)|X)) in bits (PAPER.md:130 'entropy function of M(Y)')."""
    sigma_n = 1.0 / math.sqrt(gamma)
    e = _edges(m, delta)
    sy = math.sqrt(1.0 + sigma_n ** 2)
    cdf = np.concatenate([[0.0], special.ndtr(e / sy), [1.0]])
    h_y = float(_H(np.diff(cdf)))
    x, w = _xgrid(npts)
    P = _bin_probs_given_x(x, e, sigma_n)
    h_y_x = float(np.sum(w * _H(P, axis=1)))
    return h_y, h_y_x


def mutual_info_quantised(gamma: float, m: int, delta: float) -> float:
    """I(M(Y);X) = Pi(M(Y)) - Pi(M(Y)|X)."""
    a, b = entropies(gamma, m, delta)
    return a - b


def optimal_delta(gamma: float, m: int, lo: float = 0.01, hi: float = 2.0) -> float:
    """Quantiser step maximising I(M(Y);X) (PAPER.md:132 'optimises beta')."""
    res = optimize.minimize_scalar(lambda d: -mutual_info_quantised(gamma, m, d),
                                   bounds=(lo, hi), method="bounded", options={"xatol": 1e-7})
    return float(res.x)


def slice_capacities(gamma: float, m: int, delta: float, order: Sequence[int],
                     npts: int = 4001) -> np.ndarray:
    """cap_j = 1 - H(S_j | X, S_known) in decode order (reading A-6)."""
    sigma_n = 1.0 / math.sqrt(gamma)
    e = _edges(m, delta)
    x, w = _xgrid(npts)
    P = _bin_probs_given_x(x, e, sigma_n)          # [x][b]
    b = np.arange(2 ** m)
    g = b ^ (b >> 1)
    caps = np.zeros(m)
    known = []
    h_prev = 0.0
    for j in order:
        known.append(j)
        # joint distribution of (bits in `known`) given x
        key = np.zeros_like(g)
        for t, jj in enumerate(known):
            key |= ((g >> jj) & 1) << t
        Pk = np.zeros((len(x), 2 ** len(known)))
        for kk in range(2 ** len(known)):
            Pk[:, kk] = P[:, key == kk].sum(axis=1)
        h = float(np.sum(w * _H(Pk, axis=1)))
        caps[j] = 1.0 - (h - h_prev)
        h_prev = h
    return caps


def biawgn_capacity(sigma: float) -> float:
    """Capacity of the binary-input AWGN channel (bits), y = +-1 + N(0, sigma^2)."""
    def f(y):
        p = stats.norm.pdf(y, 1.0, sigma)
        return p * np.log2(2.0 / (1.0 + np.exp(-2.0 * y / sigma ** 2)))
    val, _ = integrate.quad(f, -1 - 12 * sigma, 1 + 12 * sigma, limit=200)
    return float(val)
