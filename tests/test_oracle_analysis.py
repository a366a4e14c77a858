"""Oracle analysis formulas pinned to the paper's printed settings and SURVEY App. A values."""
import math

import numpy as np
import pytest

from cvsr_inputs import configs
from oracle import analysis as A

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
            assert s.rate <= 0.9 * caps[s.j] + 1e-3   # rate at or below 0.9 cap


def test_c1_biawgn_capacity():
    """A-16: BI-AWGN at E_b/N_0 = 1.5 dB, sigma = 0.841395: capacity 0.6023 > R = 0.5."""
    from cvsr_inputs.awgn import biawgn_sigma
    s = biawgn_sigma(0.5, 1.5)
    assert abs(s - 0.841395) < 1e-6
    assert abs(A.biawgn_capacity(s) - 0.6023) < 2e-4
