"""Host analysis formulas (paper_2108_08418_b200.keyrate) pinned to the paper's printed settings and SURVEY App. A values."""
import math

import numpy as np
import pytest

from cvsr_inputs import configs
from paper_2108_08418_b200 import keyrate as A

EPS = 2.5e-10   # PAPER.md:334 standard settings eps_EC


def test_standard_settings_snr_iab():
    """eq: SNR at the standard settings: gamma = 2.21468, I_AB = 0.84234."""
    g = A.snr(5, 0.9, 0.0186, 0.0133)
    assert abs(g - 2.214676) < 1e-6
    assert abs(A.i_ab(g) - 0.842337) < 1e-6
    # SPEC.md examples (trivial identities)
    assert A.snr(2, 1, 0, 0) == 1.0 and A.i_ab(1.0) == 0.5 and A.i_ab(3.0) == 1.0


def test_dispersion_cfinite_betafinite():
    g = A.snr(5, 0.9, 0.0186, 0.0133)
    assert abs(A.dispersion(g, EPS) - 220.765) < 1e-3
    assert abs(A.q_inv(1.25e-10) - 6.32698) < 1e-5  # not SPEC's 6.44
    assert abs(A.c_finite(g, 3.6e7, EPS) - 0.826936) < 2e-6
    assert abs(A.beta_finite(g, 3.6e7, EPS) - 0.981716) < 2e-6
    # C_Finite increases with N_R (eq: BetaFinite discussion)
    assert A.c_finite(g, 1e5, EPS) < A.c_finite(g, 1e6, EPS) < A.c_finite(g, 3.6e7, EPS) < A.i_ab(g)


def test_beta_identity_eq2_eq7():
    """equation: beta == equation: beta2."""
    rates = [0.0, 0.0, 0.15, 0.583, 0.442]
    for pi in (4.5272, 3.9):
        assert abs(A.beta(pi, 5, rates, 2.2) - A.beta2(pi, 5, rates, 2.2)) < 1e-14


def test_slepian_wolf_chain():
    """1 >= I(M(Y);X)/I_AB (data processing)."""
    for g, m in ((2.214676, 5), (1.0, 4), (0.5, 3)):
        d = A.optimal_delta(g, m)
        assert A.mutual_info_quantised(g, m, d) <= A.i_ab(g) + 1e-9


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_config_delta_is_optimal(name):
    """Configured delta* (DERIVED, parity unpinned vs paper) re-derived by the oracle."""
    cfg = configs.CONFIGS[name]
    d = A.optimal_delta(cfg.gamma, cfg.m)
    assert abs(d - cfg.delta) < 2e-4
    caps = A.slice_capacities(cfg.gamma, cfg.m, cfg.delta, cfg.order)
    for s in cfg.slices:
        if s.kind != "disclosed":
            # C2: at or below 0.9 cap; C4: the back-off ladder from the rate closest
            # to capacity in steps of 0.05 (reading R-2')
            assert s.rate < caps[s.j]
            if name == "C2":
                assert s.rate <= 0.9 * caps[s.j] + 1e-3
            else:
                k = (int(1000 * caps[s.j]) / 1000 - s.rate) / 0.05
                assert abs(k - round(k)) < 1e-6


def test_c1_biawgn_capacity():
    """A-16: BI-AWGN at E_b/N_0 = 1.5 dB, sigma = 0.841395: capacity 0.6023 > R = 0.5."""
    from cvsr_inputs.awgn import biawgn_sigma
    s = biawgn_sigma(0.5, 1.5)
    assert abs(s - 0.841395) < 1e-6
    assert abs(A.biawgn_capacity(s) - 0.6023) < 2e-4


# ----------------------------------------------------------------- NEXT-1: complexity, GA DE, key rate, N_R*
def test_ops_per_iteration_regular_equals_7G():
    """eq: EP: for a regular (dv, dc) code the degree-distribution form equals 7 G, G = dv N_R."""
    for dv, dc in ((3, 6), (4, 8), (3, 4)):
        assert abs(A.ops_per_iteration_dd(1e6, {dv: 1.0}, {dc: 1.0}) - 7 * dv * 1e6) < 1e-3
        assert A.ops_per_iteration(dv * 10 ** 6) == 7 * dv * 10 ** 6
    assert A.delta_t_model(2.0, [3.0, 5.0], [10, 1]) == 70.0


def test_phi_approximation_and_inverse():
    """eq:phiFunc approximation: phi(0) = 1, decreasing, inverse round-trips;
    close to the exact phi (numerical integral of the printed definition) for 1 <= v <= 10."""
    v = np.array([0.5, 1.0, 2.0, 5.0, 10.0, 30.0])
    w = A.phi_approx(v)
    assert A.phi_approx(0.0) == 1.0 and np.all(np.diff(w) < 0)
    assert np.allclose(A.phi_inv_approx(w), v, rtol=1e-9)
    assert A.phi_inv_approx(1.0) == 0.0
    from scipy import integrate
    for vv in (1.0, 3.0, 10.0):
        f = lambda u: np.tanh(u / 2) * np.exp(-(u - vv) ** 2 / (4 * vv))  # noqa: E731
        exact = 1 - integrate.quad(f, vv - 40 * np.sqrt(vv), vv + 40 * np.sqrt(vv))[0] / np.sqrt(4 * np.pi * vv)
        assert abs(float(A.phi_approx(vv)) - exact) / exact < 0.05


def test_ga_threshold_regular_36():
    """Textbook value: the Gaussian-approximation threshold of the (3,6) ensemble on the BI-AWGN
    channel is sigma = 0.8747 (Chung, Forney, Richardson, Urbanke 2001), below the exact BP
    threshold 0.8809 (Richardson-Urbanke)."""
    s = A.ga_threshold_sigma({3: 1.0}, {6: 1.0})
    assert abs(s - 0.8747) < 2e-3 and s < 0.8809


def test_ga_threshold_irregular_rate_half():
    """Textbook value with lambda_2 > 0: the rate-1/2 ensemble lambda = 0.30013 x + 0.28395 x^2 +
    0.41592 x^7, rho = 0.22919 x^5 + 0.77081 x^6 has the exact-DE BI-AWGN threshold sigma* =
    0.9158 (Richardson, Shokrollahi, Urbanke 2001); the GA lands within 1.5 %."""
    s = A.ga_threshold_sigma({2: 0.30013, 3: 0.28395, 8: 0.41592}, {6: 0.22919, 7: 0.77081}, iters=1000)
    assert abs(s / 0.9158 - 1) < 0.015


def test_biawgn_capacity_limits():
    """BI-AWGN capacity: -> 1 for sigma -> 0, ~ 1/(2 sigma^2 ln 2) for large sigma, 0.5 at the
    Shannon limit sigma = 0.9787 of rate 1/2; the inverse round-trips."""
    assert abs(A.biawgn_capacity(0.2) - 1.0) < 1e-5
    assert abs(A.biawgn_capacity(0.9787) - 0.5) < 2e-4
    s = 20.0
    assert abs(A.biawgn_capacity(s) / (1 / (2 * s * s * np.log(2))) - 1) < 0.01
    assert abs(A.biawgn_sigma_for_capacity(0.3414) - 1.277) < 2e-3
    assert abs(A.biawgn_capacity(A.biawgn_sigma_for_capacity(0.1)) - 0.1) < 1e-9


def test_ga_iterations_monotone():
    """eq:rob2: D_j decreases as the channel improves and is 'never' above the threshold."""
    lam, rho = {3: 1.0}, {6: 1.0}
    d = [A.ga_iterations(2.0 / s ** 2, lam, rho, 1e-6, 500) for s in (0.5, 0.7, 0.8, 0.85)]
    assert d == sorted(d) and d[0] >= 1
    assert A.ga_iterations(2.0 / 0.9 ** 2, lam, rho, 1e-6, 300) == 301


def test_key_rate_standard_settings():
    """Standard settings: eps_EC = 2 eps_s = eps_PA = eps_PE = 2.5e-10 gives the
    eps = 1e-9 of the paper's footnote; Delta_AEP = 419.53;
    K_Finite <= K at beta = 1 (C_Finite <= I_AB); K' = N_o K / Delta t."""
    e = A.eps_total(EPS, EPS / 2, EPS, EPS)
    assert abs(e - 1e-9) < 1e-24
    d = A.delta_aep(5, 1e9, EPS / 2, e)
    assert abs(d - 419.53) < 0.01
    g = A.snr(5, 0.9, 0.0186, 0.0133)
    kf = A.k_finite(1e9, 2e9, g, 1e6, EPS, 0.6721, d, EPS)
    k1 = A.key_rate(1e9, 2e9, A.i_ab(g), 0.6721, d, EPS)
    assert 0 < kf < k1
    assert A.k_prime(2e9, kf, 10.0) == 2e9 * kf / 10.0


def test_optimal_nr_is_the_argmax():
    """eq:diff_eq root == argmax of eq:simplifiedOpt by dense search, and K' is concave there
    (eq:2diff_eq claim); with S_BE = 0.6721 the optimum is N_R ~ 7.8e5 (the
    paper's 3.6e7 does not reproduce from its printed formulas: parity unpinned vs paper)."""
    g = A.snr(5, 0.9, 0.0186, 0.0133)
    e = A.eps_total(EPS, EPS / 2, EPS, EPS)
    B1 = A.b1(1e9, 0.6721, A.delta_aep(5, 1e9, EPS / 2, e), EPS)
    nr = A.optimal_nr(1e9, g, EPS, B1)
    grid = np.geomspace(1e5, 1e9, 4001)
    kp = np.array([A.kprime_of_nr(x, 1e9, g, EPS, B1, 1.0) for x in grid])
    assert abs(np.log(nr / grid[np.argmax(kp)])) < 0.01
    assert abs(nr / 7.8e5 - 1) < 0.01
    h = nr * 1e-3
    f = [A.kprime_of_nr(nr + k * h, 1e9, g, EPS, B1, 1.0) for k in (-1, 0, 1)]
    assert f[0] + f[2] - 2 * f[1] < 0


def test_slice_capacities_chain_rule():
    """Chain rule: sum_j cap_j = sum_j (1 - H(S_j | X, S_known)) = m - Pi(M(Y)|X), for any decode order."""
    for g, m in ((2.214676, 5), (1.0, 4)):
        d = A.optimal_delta(g, m)
        _, h_yx = A.entropies(g, m, d)
        for order in (list(range(m)), list(range(m))[::-1]):
            caps = A.slice_capacities(g, m, d, order)
            assert abs(caps.sum() - (m - h_yx)) < 1e-9
