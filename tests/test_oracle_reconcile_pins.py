"""Pins of the oracle's multi-stage driver O6 (`orc_reconcile`, SURVEY.md §8(c) O6;
PAPER.md:114 steps 4-6, Fig. 3) for BOTH BP schedules (flooding O5 = reading A-8,
row-layered O5' = reading R-9).  CPU only.

Each pin checks O6 against something other than itself:
* the conditioning on already-known slices, against the two-bin closed form of
  the slice LLR (scipy log_ndtr) pushed through a code whose decoder output is a
  closed-form function of the LLRs (one degree-2 check);
* the "later slices are not attempted" rule (reading A-13) with syndromes that no
  vector satisfies;
* noiseless input: Alice's labels are Bob's with D = 0 on every coded slice;
* a one-slice reconcile equals the single-slice decoder on the slice LLR.
"""
import numpy as np
import pytest
from scipy import special

import oracle
from cvsr_inputs import codes
from cvsr_inputs.quantiser import edge_table
import _brute

SCHEDULES = ("flooding", "layered")


def _bob_labels(edges: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Independent quantiser (numpy right-searchsorted = #{k: y >= e_k}) + binary-reflected Gray."""
    b = np.searchsorted(edges.astype(np.float32), y.astype(np.float32), side="right")
    return (b ^ (b >> 1)).astype(np.uint8)


def _logp_bin(e64: np.ndarray, x: float, sigma: float, b: int) -> float:
    """log P(bin b | x) = log(Phi(hi) - Phi(lo)), evaluated on the tail side with log_ndtr."""
    nb = len(e64) + 1
    lo = -np.inf if b == 0 else (e64[b - 1] - x) / sigma
    hi = np.inf if b == nb - 1 else (e64[b] - x) / sigma
    if lo > 0:
        a = special.log_ndtr(-lo)
        c = special.log_ndtr(-hi) if np.isfinite(hi) else -np.inf
    else:
        a = special.log_ndtr(hi) if np.isfinite(hi) else 0.0
        c = special.log_ndtr(lo) if np.isfinite(lo) else -np.inf
    return float(a + np.log1p(-np.exp(c - a)))


def _pair_code():
    """n = 2, one check {0, 1}: the decoder's output is a closed-form function of (L0, L1, s)."""
    return codes.from_dense(np.array([[1, 1]], np.uint8))


@pytest.mark.parametrize("schedule", SCHEDULES)
@pytest.mark.parametrize("order", [(0, 1), (1, 0)])
def test_reconcile_conditioning_closed_form(schedule, order):
    """m = 2: the first slice in `order` is disclosed, the second coded with the pair code.
    Given Bob's disclosed bit kappa the coded slice's LLR is the two-bin closed form
    L = ln P_{b0}(x) - ln P_{b1}(x) over the bins whose Gray label has the known bit = kappa
    (PAPER.md:114 step 4, reading A-2).  BP on one degree-2 check is exact:
      [L < 0] satisfies the syndrome  => D = 0, bits = [L < 0];
      otherwise                        => D = 1, post_v = L_v + (1 - 2s) L_other, bits = [post < 0].
    A conditioning mistake (wrong or no known mask, Alice's instead of Bob's bits, wrong slice)
    flips decisions on a large fraction of the frames."""
    m, delta, gamma = 2, 0.6, 1.5
    sigma = 1.0 / np.sqrt(gamma)
    e = edge_table(m, delta)
    e64 = e.astype(np.float64)
    rng = np.random.default_rng(11 + order[0])
    F = 600
    x = rng.normal(0, 1, (F, 2)).astype(np.float32)
    y = (x + rng.normal(0, sigma, x.shape)).astype(np.float32)
    lab = _bob_labels(e, y)
    jd, jc = order
    code = _pair_code()
    cl = [None, None]
    cl[jc] = code
    synd = [None, None]
    synd[jd] = _brute.pack_bits(((lab >> jd) & 1).astype(np.uint8))
    s_par = (((lab[:, 0] >> jc) & 1) ^ ((lab[:, 1] >> jc) & 1)).astype(np.uint8)
    synd[jc] = _brute.pack_bits(s_par[:, None])
    lab_a, ok, it = oracle.reconcile(cl, order, e, sigma, x, synd, max_iter=10, schedule=schedule)
    g = np.arange(4) ^ (np.arange(4) >> 1)
    checked = 0
    for f in range(F):
        L = np.empty(2)
        for v in range(2):
            kappa = (int(lab[f, v]) >> jd) & 1
            cand = [b for b in range(4) if ((g[b] >> jd) & 1) == kappa]
            b0 = [b for b in cand if not (g[b] >> jc) & 1][0]
            b1 = [b for b in cand if (g[b] >> jc) & 1][0]
            L[v] = np.clip(_logp_bin(e64, float(x[f, v]), sigma, b0) - _logp_bin(e64, float(x[f, v]), sigma, b1),
                           -40, 40)
        hard = (L < 0).astype(np.uint8)
        if (hard[0] ^ hard[1]) == s_par[f]:
            exp_bits, exp_d, margin = hard, 0, np.min(np.abs(L))
        else:
            sg = 1.0 - 2.0 * s_par[f]
            post = np.array([L[0] + sg * L[1], L[1] + sg * L[0]])
            exp_bits, exp_d, margin = (post < 0).astype(np.uint8), 1, np.min(np.abs(post))
        assert it[f, jd] == 0 and ok[f] == 1
        assert np.array_equal((lab_a[f] >> jd) & 1, (lab[f] >> jd) & 1)
        if margin < 1e-9:  # a tie decided by rounding order: not a pin
            continue
        checked += 1
        assert it[f, jc] == exp_d, (f, L, s_par[f])
        assert np.array_equal((lab_a[f] >> jc) & 1, exp_bits), (f, L, s_par[f])
    assert checked >= F - 2
    # the pin is sharp: conditioning on the wrong value of the known bit changes many decisions
    wrong = 0
    for f in range(F):
        kap = 1 - ((lab[f] >> jd) & 1)
        Lw = []
        for v in range(2):
            cand = [b for b in range(4) if ((g[b] >> jd) & 1) == kap[v]]
            b0 = [b for b in cand if not (g[b] >> jc) & 1][0]
            b1 = [b for b in cand if (g[b] >> jc) & 1][0]
            Lw.append(_logp_bin(e64, float(x[f, v]), sigma, b0) - _logp_bin(e64, float(x[f, v]), sigma, b1))
        hw = (np.array(Lw) < 0).astype(np.uint8)
        wrong += int(not np.array_equal(hw, (lab_a[f] >> jc) & 1))
    assert wrong > F // 10


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_reconcile_forced_failure_skips_later_slices(schedule):
    """Reading A-13: a frame whose slice fails stops there -- later slices are not attempted
    (iters = -1, label bits 0) and frame_ok = 0; the failed slice reports D = max_iter.
    Slice 0's code has two identical rows; frames whose two syndrome bits differ are
    unsatisfiable, the others decode."""
    m, n, max_iter = 3, 64, 7
    rng = np.random.default_rng(5)
    base = codes.regular(n, 3, 6, seed=7)
    H = base.dense()
    H0 = np.vstack([H[:1], H])  # rows 0 and 1 identical
    c0 = codes.from_dense(H0)
    c1 = codes.regular(n, 3, 6, seed=8)
    c2 = codes.regular(n, 3, 6, seed=9)
    e = edge_table(m, 0.5)
    F = 40
    x = rng.normal(0, 1, (F, n)).astype(np.float32)
    y = x.copy()  # noiseless: every satisfiable slice decodes at D = 0
    lab = _bob_labels(e, y)
    synd = [oracle.syndrome(c, lab, j) for j, c in enumerate((c0, c1, c2))]
    bad = np.arange(F) % 2 == 1
    s0 = _brute.unpack_bits(synd[0], c0.m_checks)
    s0[bad, 1] ^= 1
    synd[0] = _brute.pack_bits(s0)
    lab_a, ok, it = oracle.reconcile([c0, c1, c2], (0, 1, 2), e, 1e-6, x, synd, max_iter=max_iter,
                                     schedule=schedule)
    assert np.array_equal(ok, (~bad).astype(np.uint8))
    assert (it[bad, 0] == max_iter).all() and (it[bad, 1:] == -1).all()
    assert ((lab_a[bad] >> 1) == 0).all()
    assert (it[~bad] == 0).all()
    assert np.array_equal(lab_a[~bad], lab[~bad])


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_reconcile_noiseless_equals_bob_at_d0(schedule):
    """Noiseless channel (y = x, sigma_n -> 0, points away from bin edges): every coded
    slice's conditional LLR saturates with Bob's bit as its sign, so [L < 0] already satisfies
    the syndrome: D = 0 everywhere and Alice's labels are Bob's."""
    m, n = 5, 120
    delta = 0.3
    e = edge_table(m, delta)
    rng = np.random.default_rng(17)
    F = 12
    b = rng.integers(0, 2 ** m, (F, n))
    centre = np.concatenate([[e[0] - delta / 2], (e[:-1] + e[1:]) / 2, [e[-1] + delta / 2]])
    x = (centre[b] + rng.uniform(-0.3 * delta, 0.3 * delta, b.shape)).astype(np.float32)
    lab = _bob_labels(e, x)
    assert np.array_equal(lab, (b ^ (b >> 1)).astype(np.uint8))
    cl = [None, codes.regular(n, 3, 6, seed=1), None, codes.irregular_rate(n, 0.4, seed=2),
          codes.regular(n, 3, 6, seed=3)]
    synd = [_brute.pack_bits(((lab >> j) & 1).astype(np.uint8)) if c is None else oracle.syndrome(c, lab, j)
            for j, c in enumerate(cl)]
    for order in ((0, 1, 2, 3, 4), (4, 3, 2, 1, 0)):
        lab_a, ok, it = oracle.reconcile(cl, order, e, 1e-7, x, synd, schedule=schedule)
        assert ok.all() and (it == 0).all()
        assert np.array_equal(lab_a, lab)


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_reconcile_one_slice_equals_decoder(schedule):
    """m = 1 (sign slice): reconcile = the single-slice decoder of the same schedule on the
    unconditioned slice LLR (O4 with K = {}), bit for bit, with the same D and flags."""
    n, F = 504, 16
    code = codes.regular(n, 3, 6, seed=4)
    e = edge_table(1, 0.0)
    gamma = 6.0  # a mix of converging and failing frames
    sigma = 1.0 / np.sqrt(gamma)
    rng = np.random.default_rng(8)
    x = rng.normal(0, 1, (F, n)).astype(np.float32)
    y = (x + rng.normal(0, sigma, x.shape)).astype(np.float32)
    lab = _bob_labels(e, y)
    s = oracle.syndrome(code, lab, 0)
    lab_a, ok, it = oracle.reconcile([code], (0,), e, sigma, x, [s], max_iter=60, schedule=schedule)
    L = oracle.llr_slice(e, sigma, x, 0)
    if schedule == "flooding":
        bits, conv, d = oracle.bp_decode(code, L, s, 60)
    else:
        bits, conv, d, _ = oracle.bp_decode_layered(code, L, s, 60)
    assert np.array_equal(lab_a, _brute.unpack_bits(bits, n))
    assert np.array_equal(ok, conv) and np.array_equal(it[:, 0], d)
    assert 0 < ok.sum() < F


def test_reconcile_schedules_agree_where_both_converge():
    """Both schedules decode the same multi-stage problem to Bob's labels where they converge,
    and the layered schedule needs fewer iterations (reading R-9)."""
    m, n = 3, 1000
    e = edge_table(m, 0.5)
    gamma = 8.0
    sigma = 1.0 / np.sqrt(gamma)
    rng = np.random.default_rng(23)
    F = 16
    x = rng.normal(0, 1, (F, n)).astype(np.float32)
    y = (x + rng.normal(0, sigma, x.shape)).astype(np.float32)
    lab = _bob_labels(e, y)
    cl = [codes.irregular_rate(n, 0.1, seed=1), codes.irregular_rate(n, 0.3, seed=2),
          codes.irregular_rate(n, 0.6, seed=3)]
    synd = [oracle.syndrome(c, lab, j) for j, c in enumerate(cl)]
    la, oa, ia = oracle.reconcile(cl, (0, 1, 2), e, sigma, x, synd, schedule="flooding")
    lb, ob, ib = oracle.reconcile(cl, (0, 1, 2), e, sigma, x, synd, schedule="layered")
    both = (oa == 1) & (ob == 1)
    assert both.sum() >= F // 2
    assert np.array_equal(la[both], lab[both]) and np.array_equal(lb[both], lab[both])
    assert ib[both].sum() < ia[both].sum()
