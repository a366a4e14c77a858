"""Input generators (cvsr_inputs): construction properties, determinism, seeding."""
import numpy as np

from cvsr_inputs import awgn, codes, configs
from cvsr_inputs.quantiser import edge_table


def _no_duplicates(code):
    for c in range(code.m_checks):
        r = code.col_idx[code.row_ptr[c]:code.row_ptr[c + 1]]
        if len(np.unique(r)) != len(r) or np.any(np.diff(r) <= 0):
            return False
    return True


def test_regular_36_counts_and_determinism():
    """(3,6), n=1200 -> G=3600, rate 0.5, column histogram {3:1200}."""
    c = codes.regular(1200, 3, 6, seed=1)
    assert c.n_edges == 3600 and c.rate == 0.5
    hv, hc = codes.degree_histograms(c)
    assert hv == {3: 1200} and hc == {6: 600}
    assert _no_duplicates(c)
    assert c.digest() == codes.regular(1200, 3, 6, seed=1).digest()
    assert c.digest() != codes.regular(1200, 3, 6, seed=2).digest()


def test_irregular_degrees_rate():
    c = codes.irregular_rate(1 << 14, 0.406, seed=3)
    hv, hc = codes.degree_histograms(c)
    assert set(hv) == {2, 3, 8} and len(hc) <= 2
    assert abs(c.rate - 0.406) < 2.0 / c.n  # SPEC.md:264 realised vs design
    assert abs(c.n_edges / c.n - 3.37) < 0.01  # E/n of the PROPOSED lambda
    assert _no_duplicates(c)


def test_met_structure():
    c = codes.met_low_rate(10000, 0.04, 0.02, 3, 6, seed=5)
    hv, hc = codes.degree_histograms(c)
    assert hv[1] == 9600 and abs(c.rate - 0.02) < 1e-9
    assert hc[2] == 9600
    assert _no_duplicates(c)


def test_csc_is_permutation():
    c = codes.irregular_rate(4096, 0.5, seed=9)
    col_ptr, rows, pos = codes.csc(c)
    assert np.array_equal(np.sort(pos), np.arange(c.n_edges))
    assert np.array_equal(c.col_idx[pos], np.repeat(np.arange(c.n), np.diff(col_ptr)))


def test_awgn_frame_seeding_independent_of_batch():
    x1, y1 = awgn.quadratures(6, 100, 2.0, seed=4)
    x2, y2 = awgn.quadratures(3, 100, 2.0, seed=4, first_frame=3)
    assert np.array_equal(x1[3:], x2) and np.array_equal(y1[3:], y2)
    x, y = awgn.quadratures(64, 4096, 1.0, seed=1)
    assert abs(x.std() - 1) < 0.02 and abs((y - x).std() - 1) < 0.02


def test_configs_build():
    c2 = configs.scaled(configs.C2, 4096, 4)
    cs = c2.build_codes()
    assert cs[0] is None and cs[1] is None and cs[2] is not None
    assert len(c2.edges()) == 15 and np.array_equal(c2.edges(), edge_table(4, 0.44905))


def test_peg_construction_girth_and_degrees():
    """PEG (host C, NEXT-2): variable degrees exact, check degrees on the two target values,
    no duplicate edge, and no 4-cycle (two checks sharing two variables) -- the configuration
    model with the same degrees has some."""
    from collections import Counter

    def four_cycles(c):
        rp, ci = np.asarray(c.row_ptr), np.asarray(c.col_idx)
        pairs = Counter()
        for r in range(c.m_checks):
            vs = ci[rp[r]:rp[r + 1]]
            assert len(set(vs.tolist())) == len(vs)
            for i in range(len(vs)):
                for j in range(i + 1, len(vs)):
                    pairs[(int(vs[i]), int(vs[j]))] += 1
        return sum(v * (v - 1) // 2 for v in pairs.values())

    peg = codes.irregular_rate(4096, 0.356, seed=3, lam={2: 0.3, 3: 0.7}, construction="peg")
    cfg = codes.irregular_rate(4096, 0.356, seed=3, lam={2: 0.3, 3: 0.7})
    dv = np.bincount(np.asarray(peg.col_idx), minlength=peg.n)
    assert sorted(Counter(dv.tolist()).items()) == sorted(Counter(
        np.bincount(np.asarray(cfg.col_idx), minlength=cfg.n).tolist()).items())
    dc = np.diff(np.asarray(peg.row_ptr))
    assert set(dc.tolist()) <= {4, 5} and peg.n_edges == cfg.n_edges
    assert four_cycles(peg) == 0 and four_cycles(cfg) > 0


def test_codebook_recipes_reproduce_c4_codes():
    """The code database stores recipes + SHA digests (PAPER.md:392 database; tools/backoff.py):
    the C4 config's coded slices are exactly the codes the back-off marked good, rebuilt bit for
    bit from their recipes, and every stored trial respects the Delta R = 0.05 ladder from the
    rate closest to capacity."""
    from cvsr_inputs import codebook, configs
    entries = codebook.load()
    assert entries, "cvsr_inputs/codebook.json missing"
    cl = configs.C4.build_codes()
    for j, c in enumerate(cl):
        if c is None:
            continue
        e = codebook.good("C4", j, configs.C4.n)
        assert e is not None and e["digest"] == c.digest()
        assert e["test"]["failed"] == 0 and e["test"]["undetected"] == 0
        ladder = sorted({x["params"]["rate"] for x in entries if x["config"] == "C4" and x["slice"] == j},
                        reverse=True)
        assert abs(ladder[0] - int(1000 * e["cap"]) / 1000) < 1e-9
        assert all(abs((a - b) - 0.05) < 1e-9 for a, b in zip(ladder, ladder[1:]))
        assert e["params"]["rate"] == ladder[-1]


def test_backoff_ladder_follows_paper_procedure():
    """tools/backoff.py's ladder (reading R-2'): start at the rate closest to (not
    above) capacity, lower by Delta R = 0.05 after a failed test, MET-style below 0.1 and irregular
    first above (MET retried up to 0.25), disclose below the floor 0.01; earlier
    slices' good codes are passed to later trials.  Checked with a stand-in failure test that
    passes when R <= 0.5 cap (MET with the (3,6) core), R <= 0.7 cap with an irregular core of
    rate <= 0.4, or 0.25 < R <= 0.93 cap (irregular): the pattern measured on B200 for C4; among
    the codes passing at a rung the least decoding work wins."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("backoff", os.path.join(os.path.dirname(__file__), "..",
                                                                            "tools", "backoff.py"))
    bo = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bo)
    caps = [0.0006, 0.0022, 0.16699, 0.64855, 0.49179]  # the C4 slice capacities
    seen = []

    def trial(j, fam, r, chosen):
        seen.append((j, dict(chosen)))
        if fam == "met":
            return r <= 0.5 * caps[j], 3.0
        if fam.startswith("met_irr"):  # 0.3 / 0.35 / 0.4 pass, 0.35 with the least work
            rc = float(fam[7:])
            return rc <= 0.4 and r <= 0.7 * caps[j], {0.3: 2.0, 0.35: 1.0, 0.4: 1.5}.get(rc, 9.0)
        return 0.25 < r <= 0.93 * caps[j], 1.0

    chosen, trials = bo.ladder([0, 1, 2, 3, 4], caps, trial)
    assert chosen[0] is None and chosen[1] is None
    t2 = [(t[1], t[2], t[3]) for t in trials if t[0] == 2]
    assert [t for t in t2 if t[1] == 0.166] == [("irregular", 0.166, False), ("met_irr0.3", 0.166, False),
                                                 ("met_irr0.35", 0.166, False), ("met_irr0.4", 0.166, False),
                                                 ("met_irr0.5", 0.166, False), ("met", 0.166, False)]
    assert [t for t in t2 if t[1] == 0.116 and t[2]] == [("met_irr0.3", 0.116, True), ("met_irr0.35", 0.116, True),
                                                         ("met_irr0.4", 0.116, True)]
    assert chosen[2] == ("met_irr0.35", 0.116) and min(t[1] for t in t2) == 0.116
    assert [(t[2], t[3]) for t in trials if t[0] == 3] == [(0.648, False), (0.598, True)]
    assert chosen[4] == ("irregular", 0.441)
    assert seen[-1][1][3] == ("irregular", 0.598) and seen[-1][1][2] == ("met_irr0.35", 0.116)
