"""Host-side analysis of the paper in fp64: efficiency, finite-length rate,
complexity model, finite-key rate and the N_R optimiser.

Not part of the GPU hot path: these formulas turn the path's measured numbers
(throughput, iterations, realised code rates) into the paper's figures of
merit (beta, K, K' in bits/s).  Each function restates one PAPER.md equation,
cited by its LaTeX label.  Quantised entropies use numerical integration over
Alice's x (reading A-5: x ~ N(0,1), y = x + n, n ~ N(0, 1/gamma)).
Pinned in tests/test_keyrate.py against the paper's printed settings, closed
forms and textbook values.
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
        return p * (1.0 - np.logaddexp(0.0, -2.0 * y / sigma ** 2) / math.log(2.0))
    val, _ = integrate.quad(f, -1 - 12 * sigma, 1 + 12 * sigma, limit=200)
    return float(val)


# ---------------------------------------------------------------- complexity model (Section III.C)

def ops_per_iteration_dd(n_r: float, lam: dict, rho: dict) -> float:
    """eq: EP second line from edge-perspective degree distributions:
    E = 7 N_R (sum_b rho_b / b) / (sum_a lam_a / a) * (sum_b b rho_b).  Equals 7 G for regular codes."""
    s_rho = sum(r / b for b, r in rho.items())
    s_lam = sum(l / a for a, l in lam.items())
    return 7.0 * n_r * s_rho / s_lam * sum(b * r for b, r in rho.items())


def delta_t_model(c_h: float, E: Sequence[float], D: Sequence[float]) -> float:
    """eq:DeltaT: Delta t = c_h sum_j E_j D_j."""
    return c_h * float(sum(e * d for e, d in zip(E, D)))


# ---------------------------------------------------------------- Gaussian-approximation DE (D_j)

def phi_approx(v):
    """Approximation of eq:phiFunc: exp(-0.4527 v^0.86 + 0.0218), phi(0) = 1.
    Clipped to <= 1 (the fit exceeds 1 for v < 0.0118)."""
    v = np.asarray(v, dtype=np.float64)
    out = np.where(v > 0, np.exp(-0.4527 * np.power(np.maximum(v, 1e-300), 0.86) + 0.0218), 1.0)
    return np.minimum(out, 1.0)


def phi_inv_approx(w):
    """Inverse of the approximation: ((ln w - 0.0218) / -0.4527)^(1/0.86), 0 at w >= 1."""
    w = np.asarray(w, dtype=np.float64)
    wc = np.clip(w, 1e-300, 1.0)
    val = np.power(np.maximum((np.log(wc) - 0.0218) / -0.4527, 0.0), 1.0 / 0.86)
    return np.where(w >= 1.0, 0.0, val)


def ga_check_means(m0: float, lam: dict, rho: dict, iters: int) -> np.ndarray:
    """Mean of the check-to-variable LLR after k = 1..iters flooding iterations under the
    Gaussian approximation (reading A-19 of SURVEY §8(c): eq:rob's "log gamma" is the channel
    LLR mean m0, the recursion runs on means):
        m_c^k = sum_b rho_b phi^-1(1 - [1 - sum_a lam_a phi(m0 + (a - 1) m_c^(k-1))]^(b - 1)),  m_c^0 = 0."""
    out = np.zeros(iters)
    mc = 0.0
    for k in range(iters):
        s = sum(l * float(phi_approx(m0 + (a - 1) * mc)) for a, l in lam.items())
        # 1 - (1 - s)^(b-1) without cancellation (s falls far below 1e-16 once decoding succeeds)
        mc = sum(r * float(phi_inv_approx(-math.expm1((b - 1) * math.log1p(-s)))) for b, r in rho.items())
        out[k] = mc
    return out


def ga_ber(m0: float, lam: dict, mc: float) -> float:
    """Bit error rate of the decision after an iteration whose check means are mc: posterior of a
    degree-a variable ~ N(m0 + a mc, 2 (m0 + a mc)), node-perspective degree mix."""
    node = {a: l / a for a, l in lam.items()}
    z = sum(node.values())
    return float(sum(w / z * stats.norm.sf(math.sqrt((m0 + a * mc) / 2.0)) for a, w in node.items()))


def ga_iterations(m0: float, lam: dict, rho: dict, eps: float, max_iter: int = 1000) -> int:
    """eq:rob2: D = min {k : q_k <= eps}; max_iter + 1 if never reached."""
    for k, mc in enumerate(ga_check_means(m0, lam, rho, max_iter), start=1):
        if ga_ber(m0, lam, mc) <= eps:
            return k
    return max_iter + 1


def ga_threshold_sigma(lam: dict, rho: dict, lo: float = 0.3, hi: float = 2.0, iters: int = 2000,
                       ber_target: float = 1e-10) -> float:
    """Largest BI-AWGN noise sigma (m0 = 2 / sigma^2) for which the GA decision error falls
    below ber_target within `iters` iterations.  (With lam_2 > 0 and the printed phi fit the
    check mean settles at a large but finite value instead of diverging, so the criterion is
    the bit error rate, not the mean.)"""
    def ok(sig):
        m0 = 2.0 / sig ** 2
        return ga_ber(m0, lam, ga_check_means(m0, lam, rho, iters)[-1]) <= ber_target
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if ok(mid) else (lo, mid)
    return lo


# ---------------------------------------------------------------- finite-key rate (Section IV)

def eps_total(eps_ec: float, eps_s: float, eps_pa: float, eps_pe: float) -> float:
    """epsilon = eps_EC + 2 eps_s + eps_PA + eps_PE."""
    return eps_ec + 2.0 * eps_s + eps_pa + eps_pe


def delta_aep(m: int, N: float, eps_s: float, eps: float) -> float:
    """eq:AEP: (m+1)^2 + 4(m+1) sqrt(log2(2/eps_s^2)) + 2 log2(2/(eps^2 eps_s))
    + 4 eps_s m / (eps sqrt(N))."""
    return ((m + 1) ** 2 + 4 * (m + 1) * math.sqrt(math.log2(2.0 / eps_s ** 2))
            + 2.0 * math.log2(2.0 / (eps ** 2 * eps_s)) + 4.0 * eps_s * m / (eps * math.sqrt(N)))


def key_rate(N: float, N_o: float, beta_iab: float, s_be: float, d_aep: float, eps_pa: float) -> float:
    """eq:BPSKeyRate, bits per pulse; beta_iab = beta * I_AB.  S_BE^eps_PE is an
    input (its Holevo-bound derivation, is out of scope: SURVEY rows 37-38)."""
    return (N * (beta_iab - s_be) - math.sqrt(N) * d_aep - 2.0 * math.log2(1.0 / (2.0 * eps_pa))) / N_o


def k_finite(N: float, N_o: float, gamma: float, n_r: float, eps_ec: float, s_be: float, d_aep: float,
             eps_pa: float) -> float:
    """eq:FiniteK: eq:BPSKeyRate with beta I_AB -> C_Finite(N_R)."""
    return key_rate(N, N_o, c_finite(gamma, n_r, eps_ec), s_be, d_aep, eps_pa)


def k_prime(N_o: float, K: float, delta_t: float) -> float:
    """eq:BPSRate: K' = N_o K / Delta t, bits per second."""
    return N_o * K / delta_t


# ---------------------------------------------------------------- N_R optimisation

def b1(N: float, s_be: float, d_aep: float, eps_pa: float) -> float:
    """eq:B1: N S_BE + sqrt(N) Delta_AEP + 2 log2(1/(2 eps_PA))."""
    return N * s_be + math.sqrt(N) * d_aep + 2.0 * math.log2(1.0 / (2.0 * eps_pa))


def b2(ops_per_nr_iter: Sequence[float], D: Sequence[float], c_h: float) -> float:
    """B_2: Delta t = B_2 N_R, with ops_per_nr_iter[j] = E_j / N_R."""
    return c_h * float(sum(e * d for e, d in zip(ops_per_nr_iter, D)))


def kprime_of_nr(n_r: float, N: float, gamma: float, eps_ec: float, B1: float, B2: float) -> float:
    """eq:simplifiedOpt objective: (N C_Finite(N_R) - B_1) / (B_2 N_R)."""
    return (N * c_finite(gamma, n_r, eps_ec) - B1) / (B2 * n_r)


def dc_finite_dnr(gamma: float, n_r: float, eps_ec: float) -> float:
    """d C_Finite / d N_R of this module's eq:R_Finite (log2 in the 1/2 log N_R term)."""
    a = math.sqrt(dispersion(gamma, eps_ec)) * q_inv(eps_ec)
    return 0.5 * a * n_r ** -1.5 - 0.5 * (1.0 / math.log(2.0) - math.log2(n_r)) / n_r ** 2


def optimal_nr(N: float, gamma: float, eps_ec: float, B1: float, lo: float = 1e5, hi: float = None) -> float:
    """eq:Optimisation1 / eq:diff_eq: the stationary point of K'(N_R) in
    [lo, N] by root finding on the numerator of dK'/dN_R, N_R N C' - (N C - B_1); the better
    end point if the numerator does not change sign."""
    hi = N if hi is None else hi

    def g(x):
        return x * N * dc_finite_dnr(gamma, x, eps_ec) - (N * c_finite(gamma, x, eps_ec) - B1)
    glo, ghi = g(lo), g(hi)
    if glo > 0 and ghi < 0:
        return float(optimize.brentq(g, lo, hi, xtol=1e-6 * lo, rtol=1e-12))
    return lo if kprime_of_nr(lo, N, gamma, eps_ec, B1, 1.0) >= kprime_of_nr(hi, N, gamma, eps_ec, B1, 1.0) else hi


def biawgn_sigma_for_capacity(cap: float) -> float:
    """sigma of the BI-AWGN channel whose capacity is cap (equivalent-capacity channel for GA)."""
    return float(optimize.brentq(lambda s: biawgn_capacity(s) - cap, 0.1, 30.0, xtol=1e-10))
