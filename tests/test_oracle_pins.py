"""Pins of the fp64 oracle against what the paper and mathematics fix (CPU only).

Each test pins the oracle to something other than itself (SURVEY.md §8(c)
"What pins each part"): definitions re-derived independently, closed forms,
brute force on tiny codes, invariants and statistical bounds.
"""
import numpy as np
import pytest
from scipy import special

import oracle
from cvsr_inputs import awgn, codes
from cvsr_inputs.quantiser import edge_table
import _brute


# ----------------------------------------------------------------- quantiser (O2)

@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8])
def test_quantiser_gray_roundtrip_and_adjacency(m):
    """PAPER.md:87 Gray labelling: bin->label is a bijection and adjacent bins differ in 1 bit."""
    delta = 0.3
    e = edge_table(m, delta)
    # one representative point inside every bin
    centers = np.concatenate([[e[0] - 1.0], (e[:-1] + e[1:]) / 2, [e[-1] + 1.0]]).astype(np.float32)
    lab = oracle.quantise(e, centers)
    assert len(set(lab.tolist())) == 2 ** m
    for b in range(2 ** m - 1):
        assert bin(int(lab[b]) ^ int(lab[b + 1])).count("1") == 1
    # inverse Gray (prefix XOR) recovers the bin index
    b_rec = lab.astype(np.int64).copy()
    shift = b_rec >> 1
    while np.any(shift):
        b_rec ^= shift
        shift >>= 1
    assert np.array_equal(b_rec, np.arange(2 ** m))


def test_quantiser_ties_clamp_zero_monotone():
    m = 5
    e = edge_table(m, 0.21359)
    # ties go to the upper bin (reading A-3)
    lab_at = oracle.quantise(e, e.copy())
    lab_below = oracle.quantise(e, np.nextafter(e, np.float32(-np.inf)))
    assert np.all(lab_at != lab_below)
    # b(y) = #{k: y >= e_k} equals numpy's right-searchsorted count
    rng = np.random.default_rng(3)
    y = np.concatenate([rng.normal(0, 2, 20000), e, np.nextafter(e, np.float32(np.inf)),
                        np.nextafter(e, np.float32(-np.inf)), [0.0, -0.0, 1e30, -1e30]]).astype(np.float32)
    b = np.searchsorted(e, y, side="right")
    assert np.array_equal(oracle.quantise(e, y), (b ^ (b >> 1)).astype(np.uint8))
    # +-0 land in the upper-middle bin; +-huge clamp to outer bins
    lz = oracle.quantise(e, np.array([0.0, -0.0], np.float32))
    assert lz[0] == lz[1] == (16 ^ 8)
    lh = oracle.quantise(e, np.array([-3e38, 3e38], np.float32))
    assert lh[0] == 0 and lh[1] == (31 ^ 15)
    # monotone: bin index non-decreasing in y
    ys = np.sort(rng.normal(0, 2, 5000).astype(np.float32))
    lab = oracle.quantise(e, ys).astype(np.int64)
    bb = lab.copy()
    s = bb >> 1
    while np.any(s):
        bb ^= s
        s >>= 1
    assert np.all(np.diff(bb) >= 0)


def test_edge_table_symmetric():
    e = edge_table(5, 0.21359)
    assert np.all(np.diff(e) > 0)
    assert np.array_equal(e, -e[::-1])
    assert e[15] == 0.0


# ----------------------------------------------------------------- syndrome (O3)

def test_syndrome_bruteforce_zero_linearity():
    rng = np.random.default_rng(5)
    for trial in range(20):
        n = int(rng.integers(5, 70))
        M = int(rng.integers(1, n))
        H = (rng.random((M, n)) < 0.3).astype(np.uint8)
        H[:, 0] |= 1 - H.any(axis=1).astype(np.uint8)
        code = codes.from_dense(H)
        F = 3
        lab = rng.integers(0, 256, (F, n), dtype=np.uint8)
        for j in (0, 3, 7):
            s = oracle.syndrome(code, lab, j)
            bits = (lab >> j) & 1
            ref = (bits.astype(np.int64) @ H.T.astype(np.int64)) % 2
            assert np.array_equal(_brute.unpack_bits(s, M), ref)
        # zero -> zero, linearity
        z = oracle.syndrome(code, np.zeros((1, n), np.uint8), 0)
        assert not z.any()
        a = rng.integers(0, 2, (1, n), dtype=np.uint8)
        b = rng.integers(0, 2, (1, n), dtype=np.uint8)
        assert np.array_equal(oracle.syndrome(code, a ^ b, 0),
                              oracle.syndrome(code, a, 0) ^ oracle.syndrome(code, b, 0))


def test_slice_bits_packing():
    rng = np.random.default_rng(1)
    lab = rng.integers(0, 32, (4, 77), dtype=np.uint8)
    for j in range(5):
        w = oracle.slice_bits(lab, j)
        assert w.shape == (4, 3)
        assert np.array_equal(_brute.unpack_bits(w, 77), (lab >> j) & 1)
        assert not (w[:, 2] >> (77 - 64)).any()  # padding bits are zero


# ----------------------------------------------------------------- LLR (O4)

def test_llr_m1_closed_form():
    """m = 1 (one edge at 0): L = ln Phi(-x/sigma) - ln Phi(x/sigma)."""
    e = edge_table(1, 0.0)
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.normal(0, 3, 4000), [0.0, 8.0, -8.0, 30.0]]).astype(np.float32)
    for sigma in (0.3, 1.0, 4.4721):
        L = oracle.llr_slice(e, sigma, x, 0)
        ref = special.log_ndtr(-x.astype(np.float64) / sigma) - special.log_ndtr(x.astype(np.float64) / sigma)
        ref = np.clip(ref, -40, 40)
        assert np.max(np.abs(L - ref) / (np.abs(ref) + 1)) < 1e-12


def _bin_logp(edges64, x, sigma, b):
    """log P(bin b | x) via scipy log_ndtr differences (independent evaluation)."""
    nb = len(edges64) + 1
    lo = -np.inf if b == 0 else (edges64[b - 1] - x) / sigma
    hi = np.inf if b == nb - 1 else (edges64[b] - x) / sigma
    # P = Phi(hi) - Phi(lo) = Q(lo) - Q(hi); use the side far from the mode
    if np.isfinite(lo) and lo > 0:
        a, c = special.log_ndtr(-lo), special.log_ndtr(-hi) if np.isfinite(hi) else -np.inf
    else:
        a = special.log_ndtr(hi) if np.isfinite(hi) else 0.0
        c = special.log_ndtr(lo) if np.isfinite(lo) else -np.inf
    return a + np.log1p(-np.exp(c - a))


def test_llr_all_but_one_known_two_bins():
    """All other slices known => exactly two candidate bins: L = ln(P_b0 / P_b1)."""
    m, delta, sigma = 4, 0.44905, 1.0
    e = edge_table(m, delta)
    e64 = e.astype(np.float64)
    rng = np.random.default_rng(7)
    x = rng.normal(0, 1.5, 300).astype(np.float32)
    g = np.arange(16) ^ (np.arange(16) >> 1)
    for j in range(m):
        mask = ((1 << m) - 1) & ~(1 << j)
        kl = rng.integers(0, 16, x.shape, dtype=np.uint8)
        L = oracle.llr_slice(e, sigma, x, j, mask, kl)
        for i in range(len(x)):
            cand = [b for b in range(16) if (g[b] & mask) == (kl[i] & mask)]
            assert len(cand) == 2
            b0 = [b for b in cand if not (g[b] >> j) & 1][0]
            b1 = [b for b in cand if (g[b] >> j) & 1][0]
            ref = np.clip(_bin_logp(e64, float(x[i]), sigma, b0) - _bin_logp(e64, float(x[i]), sigma, b1), -40, 40)
            assert abs(L[i] - ref) <= 1e-9 * (abs(ref) + 1)


def test_llr_msb_antisymmetry_and_saturation():
    m, delta = 5, 0.21359
    e = edge_table(m, delta)
    rng = np.random.default_rng(11)
    x = rng.normal(0, 1, 1000).astype(np.float32)
    L1 = oracle.llr_slice(e, 0.67, x, m - 1)
    L2 = oracle.llr_slice(e, 0.67, -x, m - 1)
    assert np.max(np.abs(L1 + L2)) < 1e-12
    # noiseless saturation: x at a bin centre, tiny sigma
    centers = ((np.arange(32) - 16) + 0.5) * delta
    lab = oracle.quantise(e, centers.astype(np.float32))
    for j in range(m):
        L = oracle.llr_slice(e, 1e-3, centers.astype(np.float32), j)
        assert np.all(np.abs(L) == 40.0)
        assert np.array_equal(L < 0, ((lab >> j) & 1).astype(bool))


def test_llr_monte_carlo_posterior():
    """Conditional LLR matches an empirical posterior: bucket x, count l_j."""
    m, gamma = 5, 2.214676
    delta = 0.21359
    sigma = 1 / np.sqrt(gamma)
    e = edge_table(m, delta)
    rng = np.random.default_rng(2021)
    N = 2_000_000
    x = rng.normal(0, 1, N)
    y = (x + sigma * rng.normal(0, 1, N)).astype(np.float32)
    x = x.astype(np.float32)
    lab = oracle.quantise(e, y)
    j = 3
    known = 0b00111  # LSB-first: slices 0..2 known
    sel = (np.abs(x - 0.3) < 0.01) & ((lab & known) == 0b101)
    assert sel.sum() > 200
    p1 = ((lab[sel] >> j) & 1).mean()
    L = oracle.llr_slice(e, sigma, x[sel], j, known, lab[sel])
    p1_pred = np.mean(1 / (1 + np.exp(L)))
    se = np.sqrt(p1_pred * (1 - p1_pred) / sel.sum())
    assert abs(p1 - p1_pred) < 4 * se + 0.01


def test_llr_biawgn_closed_form():
    y = np.array([-30, -1.0, 0.0, 0.5, 3.0, 30], np.float32)
    L = oracle.llr_biawgn(y, 0.707946)
    assert np.allclose(L, np.clip(2 * y.astype(np.float64) / 0.707946, -40, 40), rtol=0, atol=1e-12)


# ----------------------------------------------------------------- BP (O5)

def test_bp_tree_exact_marginals():
    """Cycle-free Tanner graphs: BP posteriors equal brute-force MAP marginals (theorem)."""
    rng = np.random.default_rng(12)
    worst = 0.0
    for trial in range(60):
        H = _brute.random_tree_code(rng, int(rng.integers(2, 6)), 4)
        if H.shape[1] > 16:
            continue
        code = codes.from_dense(H)
        L = rng.normal(0, 3, H.shape[1])
        u = rng.integers(0, 2, H.shape[1], dtype=np.uint8)
        s = (H.astype(np.int64) @ u) % 2
        synd = _brute.pack_bits(s[None, :])
        K = 2 * H.shape[0] + 2
        c2v, post = oracle.bp_trace(code, L[None, :], synd, K)
        ref = _brute.exact_marginal_llr(H, s, L)
        worst = max(worst, np.max(np.abs(post[0] - ref) / (np.abs(ref) + 1)))
    assert worst < 1e-12


def test_bp_single_parity_check_closed_form():
    """One check of degree d, one iteration: r_e = (1-2s) 2 atanh(prod_{e'!=e} tanh(L/2))."""
    rng = np.random.default_rng(4)
    for d in (2, 3, 6, 10):
        H = np.ones((1, d), np.uint8)
        code = codes.from_dense(H)
        for s in (0, 1):
            L = rng.normal(0, 2, d)
            c2v, post = oracle.bp_trace(code, L[None, :], np.array([[s]], np.uint32), 1)
            t = np.tanh(L / 2)
            for e in range(d):
                ref = (1 - 2 * s) * 2 * np.arctanh(np.prod(np.delete(t, e)))
                assert abs(c2v[0, e] - ref) < 1e-10 * (abs(ref) + 1)
            assert np.allclose(post[0], L + c2v[0], atol=1e-12)


def test_bp_repetition_code_sum():
    """Repetition code (chain of degree-2 checks): posterior = signed sum of all LLRs."""
    n = 9
    H = np.zeros((n - 1, n), np.uint8)
    for i in range(n - 1):
        H[i, i] = H[i, i + 1] = 1
    code = codes.from_dense(H)
    rng = np.random.default_rng(9)
    L = rng.normal(0, 1.5, n)
    u = rng.integers(0, 2, n, dtype=np.uint8)
    s = (H.astype(np.int64) @ u) % 2
    c2v, post = oracle.bp_trace(code, L[None, :], _brute.pack_bits(s[None, :]), n + 1)
    sign = 1 - 2 * (u ^ u[0]).astype(np.int64)   # relative sign fixed by the syndrome
    for v in range(n):
        ref = np.sum(L * sign * sign[v])
        assert abs(post[0, v] - ref) < 1e-10


def test_bp_hamming_ml_agreement():
    """(7,4) Hamming: BP-converged output == syndrome-constrained ML on >= 99% (statistical)."""
    H = np.array([[1, 0, 1, 0, 1, 0, 1], [0, 1, 1, 0, 0, 1, 1], [0, 0, 0, 1, 1, 1, 1]], np.uint8)
    code = codes.from_dense(H)
    rng = np.random.default_rng(3)
    T = 3000
    sigma = awgn.biawgn_sigma(4 / 7, 3.0)
    u = rng.integers(0, 2, (T, 7), dtype=np.uint8)
    y = (1 - 2.0 * u) + sigma * rng.normal(0, 1, (T, 7))
    L = 2 * y / sigma ** 2
    s = (u.astype(np.int64) @ H.T) % 2
    bits, conv, iters = oracle.bp_decode(code, L, _brute.pack_bits(s), max_iter=50)
    dec = _brute.unpack_bits(bits, 7)
    agree = n_conv = 0
    for t in range(T):
        if conv[t]:
            n_conv += 1
            agree += np.array_equal(dec[t], _brute.ml_decode(H, s[t], L[t]))
    assert n_conv > 0.9 * T
    assert agree / n_conv >= 0.99


def test_bp_sign_symmetry_bit_exact():
    """decode(L*(1-2u), Hu) = u XOR decode(L, 0) with identical D."""
    code = codes.regular(504, 3, 6, seed=2)
    rng = np.random.default_rng(8)
    F = 12
    sigma = awgn.biawgn_sigma(0.5, 1.8)
    L = 2 * (1 + sigma * rng.normal(0, 1, (F, code.n))) / sigma ** 2
    u = rng.integers(0, 2, (F, code.n), dtype=np.uint8)
    s_u = oracle.syndrome(code, u, 0)
    z = np.zeros_like(s_u)
    b1, c1, d1 = oracle.bp_decode(code, L * (1 - 2.0 * u), s_u)
    b0, c0, d0 = oracle.bp_decode(code, L, z)
    assert np.array_equal(c1, c0) and np.array_equal(d1, d0)
    assert np.array_equal(_brute.unpack_bits(b1, code.n), u ^ _brute.unpack_bits(b0, code.n))


def test_bp_noiseless_and_converged_invariant():
    code = codes.regular(600, 3, 6, seed=4)
    rng = np.random.default_rng(1)
    F = 6
    u = rng.integers(0, 2, (F, code.n), dtype=np.uint8)
    s = oracle.syndrome(code, u, 0)
    L = 40.0 * (1 - 2.0 * u)
    bits, conv, iters = oracle.bp_decode(code, L, s)
    assert conv.all() and (iters == 0).all()
    assert np.array_equal(_brute.unpack_bits(bits, code.n), u)
    # noisy: every converged frame satisfies H xhat = s exactly
    sigma = awgn.biawgn_sigma(0.5, 1.2)
    Ln = 2 * ((1 - 2.0 * u) + sigma * rng.normal(0, 1, u.shape)) / sigma ** 2
    bits, conv, iters = oracle.bp_decode(code, Ln, s)
    dec = _brute.unpack_bits(bits, code.n)
    s_dec = oracle.syndrome(code, dec, 0)
    for f in range(F):
        assert conv[f] == np.array_equal(s_dec[f], s[f])


def test_bp_36_threshold_trend():
    """(3,6) BP threshold sigma* = 0.8809 (E_b/N_0 = 1.10 dB): FER falls with n above it,
    and stays ~1 below it (textbook special case; PAPER.md:371 trend)."""
    def fer(n, ebn0, F=48):
        code = codes.regular(n, 3, 6, seed=7)
        u, y = awgn.biawgn(F, n, awgn.biawgn_sigma(0.5, ebn0), seed=99)
        s = oracle.syndrome(code, u, 0)
        L = oracle.llr_biawgn(y, awgn.biawgn_sigma(0.5, ebn0) ** 2)
        _, conv, _ = oracle.bp_decode(code, L, s)
        return 1 - conv.mean()
    assert fer(4096, 2.0) < fer(256, 2.0)
    assert fer(2048, 0.3) > 0.9


# ----------------------------------------------------------------- verification hash (R-6)
def test_hash_key1_is_word_checksum():
    """key = 1: h = sum of the little-endian 32-bit words mod p (numpy '<u4' view, padding zeros)."""
    from oracle import verify
    rng = np.random.default_rng(7)
    for n in (1, 3, 4, 5, 17, 1024):
        lab = rng.integers(0, 256, size=(3, n), dtype=np.uint8)
        pad = np.zeros((3, (-n) % 4), np.uint8)
        words = np.concatenate([lab, pad], axis=1).copy().view("<u4").astype(object)
        want = [int(sum(r)) % verify.P61 for r in words]
        assert list(map(int, verify.frame_hash(lab, 1))) == want


def test_hash_key_2pow32_is_shifted_integer():
    """key = 2^32: h = 2^32 * int.from_bytes(label, 'little') mod p (exponent offset i+1, byte order)."""
    from oracle import verify
    rng = np.random.default_rng(8)
    for n in (1, 2, 7, 8, 33, 1000):
        lab = rng.integers(0, 256, size=(4, n), dtype=np.uint8)
        want = [((1 << 32) * int.from_bytes(r.tobytes(), "little")) % verify.P61 for r in lab]
        assert list(map(int, verify.frame_hash(lab, 1 << 32))) == want


def test_hash_zero_and_collision_bound():
    """Zero string hashes to 0 for every key; distinct strings differ at random keys (<= W/p collisions)."""
    from oracle import verify
    rng = np.random.default_rng(9)
    z = np.zeros((2, 37), np.uint8)
    for key in (1, 2, 12345, verify.P61 - 2):
        assert not verify.frame_hash(z, key).any()
    lab = rng.integers(0, 32, size=(1, 512), dtype=np.uint8)
    for t in range(20):
        other = lab.copy()
        other[0, rng.integers(0, 512)] ^= np.uint8(1 << rng.integers(0, 5))
        key = int(rng.integers(1, verify.P61 - 1))
        assert verify.frame_hash(lab, key)[0] != verify.frame_hash(other, key)[0]
    with pytest.raises(ValueError):
        verify.frame_hash(lab, 0)


# ----------------------------------------------------------------- Toeplitz privacy amplification (R-8)
def test_pa_equals_numpy_convolution_window():
    """y_i = (t * x)[n_in - 1 + i] mod 2: the window of numpy's integer convolution."""
    from oracle import pa
    rng = np.random.default_rng(21)
    for n_in, n_out in ((1, 1), (7, 3), (64, 64), (100, 37), (513, 200)):
        t = rng.integers(0, 2, n_in + n_out - 1, dtype=np.uint8)
        x = rng.integers(0, 2, n_in, dtype=np.uint8)
        conv = np.convolve(t.astype(np.int64), x.astype(np.int64))
        assert np.array_equal(pa.toeplitz_hash(t, x, n_out), (conv[n_in - 1: n_in - 1 + n_out] & 1).astype(np.uint8))


def test_pa_special_seeds_and_linearity():
    """Unit seed at n_in - 1 + s is a shift (y_i = x_{i-s}); the all-ones seed gives the parity of x
    in every output; y is linear in x and in t."""
    from oracle import pa
    rng = np.random.default_rng(22)
    n_in, n_out = 50, 20
    x = rng.integers(0, 2, n_in, dtype=np.uint8)
    for s in (0, 3, 19):
        t = np.zeros(n_in + n_out - 1, np.uint8)
        t[n_in - 1 + s] = 1
        want = np.array([x[i - s] if 0 <= i - s < n_in else 0 for i in range(n_out)], np.uint8)
        assert np.array_equal(pa.toeplitz_hash(t, x, n_out), want)
    assert np.all(pa.toeplitz_hash(np.ones(n_in + n_out - 1, np.uint8), x, n_out) == x.sum() % 2)
    t1, t2 = (rng.integers(0, 2, n_in + n_out - 1, dtype=np.uint8) for _ in range(2))
    x2 = rng.integers(0, 2, n_in, dtype=np.uint8)
    assert np.array_equal(pa.toeplitz_hash(t1, x ^ x2, n_out), pa.toeplitz_hash(t1, x, n_out) ^ pa.toeplitz_hash(t1, x2, n_out))
    assert np.array_equal(pa.toeplitz_hash(t1 ^ t2, x, n_out), pa.toeplitz_hash(t1, x, n_out) ^ pa.toeplitz_hash(t2, x, n_out))
    w = pa.pack_bits(x)
    assert np.array_equal(pa.unpack_bits(w, n_in), x) and w.dtype == np.dtype("<u4")


def test_pa_two_universal():
    """2-universality: for a fixed x != 0 and a uniform seed, P(T x = 0) = 2^-n_out."""
    from oracle import pa
    from scipy import stats as st
    rng = np.random.default_rng(23)
    n_in, n_out, trials = 40, 3, 4000
    x = rng.integers(0, 2, n_in, dtype=np.uint8)
    x[5] = 1
    zeros = sum(not pa.toeplitz_hash(rng.integers(0, 2, n_in + n_out - 1, dtype=np.uint8), x, n_out).any()
                for _ in range(trials))
    ci = st.binomtest(zeros, trials).proportion_ci(0.999)
    assert ci.low <= 1 / 8 <= ci.high


# ----------------------------------------------------------------- row-layered BP (O5', reading R-9)

def test_layers_valid_and_greedy():
    """Checks of one layer share no variable; each check's layer is the smallest one not used
    by an earlier neighbouring check (brute force over pairs of rows)."""
    for code in (codes.regular(240, 3, 6, seed=5), codes.irregular_rate(300, 0.4, seed=2)):
        col = oracle.layers(code)
        H = code.dense().astype(bool)
        share = (H.astype(np.int64) @ H.T.astype(np.int64)) > 0
        M = code.m_checks
        for c in range(M):
            nb = [c2 for c2 in range(M) if c2 != c and share[c, c2]]
            assert all(col[c2] != col[c] for c2 in nb)
            earlier = {int(col[c2]) for c2 in nb if c2 < c}
            assert col[c] == min(set(range(M + 1)) - earlier)


def test_layered_tree_exact_marginals():
    """Cycle-free Tanner graphs: the layered schedule also reaches the exact MAP marginals."""
    rng = np.random.default_rng(21)
    worst = 0.0
    for trial in range(60):
        H = _brute.random_tree_code(rng, int(rng.integers(2, 6)), 4)
        if H.shape[1] > 16:
            continue
        code = codes.from_dense(H)
        L = rng.normal(0, 3, H.shape[1])
        u = rng.integers(0, 2, H.shape[1], dtype=np.uint8)
        s = (H.astype(np.int64) @ u) % 2
        K = 2 * H.shape[0] + 2
        _, _, _, post = oracle.bp_decode_layered(code, L[None, :], _brute.pack_bits(s[None, :]), K,
                                                 stop_early=False)
        ref = _brute.exact_marginal_llr(H, s, L)
        worst = max(worst, np.max(np.abs(post[0] - ref) / (np.abs(ref) + 1)))
    assert worst < 1e-12


def test_layered_repetition_chain_one_sweep():
    """Repetition chain H[i] = e_i + e_{i+1}: layers alternate even/odd checks.  With L = 0
    except L_0, one layered iteration carries L_0 (signed by the syndrome) along the chain
    only as far as the two-layer sweep reaches: variables 0..2 get it, so does every
    variable after enough iterations (posterior = signed sum, as in flooding)."""
    n = 9
    H = np.zeros((n - 1, n), np.uint8)
    for i in range(n - 1):
        H[i, i] = H[i, i + 1] = 1
    code = codes.from_dense(H)
    col = oracle.layers(code)
    assert list(col) == [i % 2 for i in range(n - 1)]
    rng = np.random.default_rng(9)
    L = rng.normal(0, 1.5, n)
    u = rng.integers(0, 2, n, dtype=np.uint8)
    s = (H.astype(np.int64) @ u) % 2
    _, _, _, post = oracle.bp_decode_layered(code, L[None, :], _brute.pack_bits(s[None, :]), n + 1,
                                             stop_early=False)
    sign = 1 - 2 * (u ^ u[0]).astype(np.int64)
    for v in range(n):
        assert abs(post[0, v] - np.sum(L * sign * sign[v])) < 1e-10


def test_layered_disjoint_checks_equal_flooding():
    """When no two checks share a variable there is one layer and the layered schedule is the
    flooding schedule: identical decisions, D and posteriors."""
    rng = np.random.default_rng(5)
    H = np.zeros((6, 30), np.uint8)
    perm = rng.permutation(30)
    for c in range(6):
        H[c, perm[5 * c:5 * c + 5]] = 1
    code = codes.from_dense(H)
    assert (oracle.layers(code) == 0).all()
    L = rng.normal(0.5, 2, (8, 30))
    u = rng.integers(0, 2, (8, 30), dtype=np.uint8)
    s = oracle.syndrome(code, u, 0)
    b1, c1, d1, p1 = oracle.bp_decode_layered(code, L, s, 3, stop_early=False)
    c2v, p2 = oracle.bp_trace(code, L, s, 3)
    assert np.allclose(p1, p2, atol=1e-12)
    b1, c1, d1, _ = oracle.bp_decode_layered(code, L, s)
    b2, c2, d2 = oracle.bp_decode(code, L, s)
    assert np.array_equal(b1, b2) and np.array_equal(c1, c2) and np.array_equal(d1, d2)


def test_layered_hamming_ml_and_fewer_iterations():
    """(7,4) Hamming: layered-converged output == ML on >= 99 %; and on a (3,6) code the
    layered schedule needs fewer mean iterations than flooding at the same frames."""
    H = np.array([[1, 0, 1, 0, 1, 0, 1], [0, 1, 1, 0, 0, 1, 1], [0, 0, 0, 1, 1, 1, 1]], np.uint8)
    code = codes.from_dense(H)
    rng = np.random.default_rng(3)
    T = 2000
    sigma = awgn.biawgn_sigma(4 / 7, 3.0)
    u = rng.integers(0, 2, (T, 7), dtype=np.uint8)
    L = 2 * ((1 - 2.0 * u) + sigma * rng.normal(0, 1, (T, 7))) / sigma ** 2
    s = (u.astype(np.int64) @ H.T) % 2
    bits, conv, iters, _ = oracle.bp_decode_layered(code, L, _brute.pack_bits(s), max_iter=50)
    dec = _brute.unpack_bits(bits, 7)
    ok = [np.array_equal(dec[t], _brute.ml_decode(H, s[t], L[t])) for t in range(T) if conv[t]]
    assert len(ok) > 0.9 * T and np.mean(ok) >= 0.99
    code = codes.regular(1008, 3, 6, seed=3)
    F = 24
    sigma = awgn.biawgn_sigma(0.5, 1.6)
    u = rng.integers(0, 2, (F, code.n), dtype=np.uint8)
    L = 2 * ((1 - 2.0 * u) + sigma * rng.normal(0, 1, u.shape)) / sigma ** 2
    s = oracle.syndrome(code, u, 0)
    _, cf, df = oracle.bp_decode(code, L, s)
    bl, cl, dl, _ = oracle.bp_decode_layered(code, L, s)
    assert cl.sum() >= cf.sum()
    both = (cf == 1) & (cl == 1)
    assert both.sum() >= F // 2 and dl[both].mean() < 0.75 * df[both].mean()
    assert np.array_equal(_brute.unpack_bits(bl, code.n)[cl == 1], u[cl == 1])
