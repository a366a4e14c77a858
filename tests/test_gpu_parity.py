"""CUDA path (libcvsr.so via the C ABI) vs the fp64 oracle on the same seeded inputs.

Parity criteria (north star): quantiser labels, slice bits
and syndromes bit-exact; LLRs and BP messages/posteriors within
|gpu - ref| <= 1e-4 (|ref| + 1) (reading A-22); decoded bits identical on
every frame where the oracle converges; FER inside the oracle's 95%
Clopper-Pearson interval.
"""
import numpy as np
import pytest
import torch
from scipy import stats

import _brute
import oracle
from cvsr_inputs import awgn, codes, configs
from cvsr_inputs.quantiser import edge_table

pytestmark = pytest.mark.gpu

TOL = 1e-4


def rel_err(a, ref):
    return float(np.max(np.abs(np.asarray(a, np.float64) - ref) / (np.abs(ref) + 1.0))) if np.size(ref) else 0.0


def dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def host_u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.fixture(scope="module")
def cv(gpu):
    from paper_2108_08418_b200 import cvsr
    return cvsr


@pytest.fixture(scope="module")
def ctx(cv):
    c = cv.cvsr_ctx_create(0, torch.cuda.current_stream())
    yield c
    cv.cvsr_ctx_destroy(c)


def load(cv, ctx, code):
    return cv.cvsr_code_load(ctx, code.n, code.m_checks, code.row_ptr, code.col_idx)


def gpu_decode(cv, ctx, code, llr32, synd, max_iter=100):
    F = llr32.shape[0]
    h = load(cv, ctx, code)
    bits = torch.empty((F, (code.n + 31) // 32), dtype=torch.int32, device="cuda")
    conv = torch.empty(F, dtype=torch.uint8, device="cuda")
    iters = torch.empty(F, dtype=torch.int32, device="cuda")
    cv.cvsr_decode(ctx, h, dev(llr32), dev(synd), F, cv.decode_opts(max_iter, 40.0), bits, conv, iters)
    cv.cvsr_ctx_sync(ctx)
    cv.cvsr_code_free(h)
    return host_u32(bits), conv.cpu().numpy(), iters.cpu().numpy()


def gpu_trace(cv, ctx, code, llr32, synd, k):
    F = llr32.shape[0]
    h = load(cv, ctx, code)
    c2v = torch.empty((F, code.n_edges), dtype=torch.float32, device="cuda")
    post = torch.empty((F, code.n), dtype=torch.float32, device="cuda")
    cv.cvsr_decode_trace(ctx, h, dev(llr32), dev(synd), F, k, 40.0, c2v, post)
    cv.cvsr_ctx_sync(ctx)
    cv.cvsr_code_free(h)
    return c2v.cpu().numpy(), post.cpu().numpy()


# ------------------------------------------------------------------ Bob side

@pytest.mark.parametrize("m,delta", [(1, 0.0), (4, 0.44905), (5, 0.21359), (8, 0.013)])
def test_quantise_bitexact(cv, ctx, m, delta):
    e = edge_table(m, delta)
    rng = np.random.default_rng(m)
    y = np.concatenate([rng.normal(0, 3, 1_000_003), e, np.nextafter(e, np.float32(np.inf)),
                        np.nextafter(e, np.float32(-np.inf)), [0.0, -0.0, 3e38, -3e38, 1e-45, -1e-45]]
                       ).astype(np.float32)
    ref = oracle.quantise(e, y)
    yd = dev(y)
    out = torch.empty(len(y), dtype=torch.uint8, device="cuda")
    q = cv.make_quantiser(e)
    cv.cvsr_quantise(ctx, q, yd, len(y), out)
    assert np.array_equal(out.cpu().numpy(), ref)
    # unaligned views (scalar path) give the same labels
    out2 = torch.empty(len(y) - 1, dtype=torch.uint8, device="cuda")
    cv.cvsr_quantise(ctx, q, yd[1:], len(y) - 1, out2)
    assert np.array_equal(out2.cpu().numpy(), ref[1:])


CODES = {
    "c1_36": lambda: codes.regular(1024, 3, 6, seed=1),
    "irreg_ragged": lambda: codes.irregular_rate(4100, 0.406, seed=3),
    "met": lambda: codes.met_low_rate(2000, 0.04, 0.02, 3, 6, seed=5),
    "high_dc": lambda: codes.regular(1500, 3, 15, seed=2),
}


@pytest.mark.parametrize("name,F", [(k, 37) for k in CODES] + [("c1_36", 300), ("c1_36", 600), ("c1_36", 1200),
                                                                  ("irreg_ragged", 1201)])
def test_slice_bits_and_syndrome_bitexact(cv, ctx, name, F):
    """Bit-exact vs the oracle; F = 300 / 600 / 1200 take the shared-memory syndrome kernel with
    2 / 4 / 8 frames per block (1201: a ragged last block), n = 4100 the unaligned pack path."""
    code = CODES[name]()
    rng = np.random.default_rng(17)
    lab = rng.integers(0, 256, (F, code.n), dtype=np.uint8)
    h = load(cv, ctx, code)
    ld = dev(lab)
    for j in (0, 2, 7):
        s = torch.empty((F, (code.m_checks + 31) // 32), dtype=torch.int32, device="cuda")
        cv.cvsr_syndrome(ctx, h, ld, F, j, s)
        assert np.array_equal(host_u32(s), oracle.syndrome(code, lab, j))
        b = torch.empty((F, (code.n + 31) // 32), dtype=torch.int32, device="cuda")
        cv.cvsr_slice_bits(ctx, ld, F, code.n, j, b)
        assert np.array_equal(host_u32(b), oracle.slice_bits(lab, j))
    cv.cvsr_code_free(h)


# ------------------------------------------------------------------ LLR

@pytest.mark.parametrize("gamma,m,delta", [(2.214676, 5, 0.21359), (1.0, 4, 0.44905), (0.08, 1, 0.0)])
def test_llr_slice_parity(cv, ctx, gamma, m, delta):
    e = edge_table(m, delta)
    sigma = float(1 / np.sqrt(gamma))
    F, n = 5, 4001
    x, y = awgn.quadratures(F, n, gamma, seed=31)
    x[0, :50] *= 4.0  # tails
    lab_bob = oracle.quantise(e, y)
    rng = np.random.default_rng(5)
    wrong = lab_bob ^ (rng.random(lab_bob.shape) < 0.1).astype(np.uint8) * rng.integers(0, 2 ** m, lab_bob.shape, dtype=np.uint8)
    q = cv.make_quantiser(e)
    xd = dev(x)
    full = (1 << m) - 1
    worst = 0.0
    for j in range(m):
        for mask, kl in ((0, None), (((1 << j) - 1), lab_bob), (full & ~(1 << j), lab_bob),
                         (full & ~(1 << j), wrong)):
            ref = oracle.llr_slice(e, sigma, x, j, mask, kl)
            out = torch.empty((F, n), dtype=torch.float32, device="cuda")
            cv.cvsr_llr_slice(ctx, q, xd, F, n, sigma, j, mask, dev(kl) if mask else None, 40.0, out)
            worst = max(worst, rel_err(out.cpu().numpy(), ref))
    assert worst <= TOL, worst


def test_llr_biawgn_parity(cv, ctx):
    sigma = awgn.biawgn_sigma(0.5, 1.5)
    u, y = awgn.biawgn(3, 1000, sigma, seed=1)
    out = torch.empty(y.shape, dtype=torch.float32, device="cuda")
    cv.cvsr_llr_biawgn(ctx, dev(y), y.size, sigma ** 2, 40.0, out)
    assert rel_err(out.cpu().numpy(), oracle.llr_biawgn(y, sigma ** 2)) <= 1e-6


# ------------------------------------------------------------------ BP messages

def _channel(code, F, ebn0, seed):
    sigma = awgn.biawgn_sigma(max(code.rate, 0.02), ebn0)
    u, y = awgn.biawgn(F, code.n, sigma, seed=seed)
    llr = np.clip(2.0 * y.astype(np.float64) / sigma ** 2, -40, 40).astype(np.float32)
    return u, llr, oracle.syndrome(code, u, 0)


@pytest.mark.parametrize("name", list(CODES))
def test_trace_messages_parity(cv, ctx, name):
    code = CODES[name]()
    ebn0 = {"met": -1.0}.get(name, 1.5)
    F = 45  # two tiles, ragged
    u, llr, synd = _channel(code, F, ebn0, seed=7)
    for k in (1, 2, 5, 10):
        c2v_ref, post_ref = oracle.bp_trace(code, llr.astype(np.float64), synd, k)
        c2v, post = gpu_trace(cv, ctx, code, llr, synd, k)
        assert rel_err(c2v, c2v_ref) <= TOL, (k, rel_err(c2v, c2v_ref))
        assert rel_err(post, post_ref) <= TOL, (k, rel_err(post, post_ref))


def test_tree_exact_marginals_gpu(cv, ctx):
    rng = np.random.default_rng(12)
    for trial in range(25):
        H = _brute.random_tree_code(rng, int(rng.integers(2, 6)), 4)
        if H.shape[1] > 16:
            continue
        code = codes.from_dense(H)
        L = rng.normal(0, 3, (3, H.shape[1]))
        u = rng.integers(0, 2, (3, H.shape[1]), dtype=np.uint8)
        s = (u.astype(np.int64) @ H.T) % 2
        _, post = gpu_trace(cv, ctx, code, L.astype(np.float32), _brute.pack_bits(s), 2 * H.shape[0] + 2)
        for f in range(3):
            ref = _brute.exact_marginal_llr(H, s[f], L[f].astype(np.float32).astype(np.float64))
            assert rel_err(post[f], ref) <= TOL


# ------------------------------------------------------------------ decode (C1)

def _clopper_pearson(k, n, a=0.05):
    lo = stats.beta.ppf(a / 2, k, n - k + 1) if k > 0 else 0.0
    hi = stats.beta.ppf(1 - a / 2, k + 1, n - k) if k < n else 1.0
    return lo, hi


def test_decode_c1_parity(cv, ctx):
    """C1: (3,6) n=1024, 100 frames, E_b/N_0 = 1.5 dB BI-AWGN (reading A-16)."""
    c = configs.C1
    code = codes.regular(c["n"], c["dv"], c["dc"], seed=configs.CODE_SEED)
    sigma = awgn.biawgn_sigma(0.5, c["ebn0_db"])
    u, y = awgn.biawgn(c["frames"], c["n"], sigma)
    llr_d = torch.empty(y.shape, dtype=torch.float32, device="cuda")
    cv.cvsr_llr_biawgn(ctx, dev(y), y.size, sigma ** 2, 40.0, llr_d)
    llr = llr_d.cpu().numpy()
    synd = oracle.syndrome(code, u, 0)
    b_ref, c_ref, i_ref = oracle.bp_decode(code, llr.astype(np.float64), synd, c["max_iter"])
    b, cg, it = gpu_decode(cv, ctx, code, llr, synd, c["max_iter"])
    conv_ok = c_ref.astype(bool)
    assert np.array_equal(b[conv_ok], b_ref[conv_ok])
    assert np.sum(cg != c_ref) <= 2
    assert np.sum(it[conv_ok] != i_ref[conv_ok]) <= 2
    k_fail = int(np.sum(c_ref == 0))
    lo, hi = _clopper_pearson(k_fail, len(c_ref))
    assert lo <= float(np.mean(cg == 0)) <= hi
    # converged => H xhat = s exactly; noiseless decoded bits match u
    dec = _brute.unpack_bits(b, code.n)
    s_dec = oracle.syndrome(code, dec, 0)
    for f in range(len(cg)):
        if cg[f]:
            assert np.array_equal(s_dec[f], synd[f])


def test_decode_determinism_and_batch_invariance(cv, ctx):
    code = codes.regular(1024, 3, 6, seed=1)
    u, llr, synd = _channel(code, 100, 1.5, seed=3)
    a = gpu_decode(cv, ctx, code, llr, synd)
    b = gpu_decode(cv, ctx, code, llr, synd)
    sub = gpu_decode(cv, ctx, code, llr[37:90], synd[37:90])
    perm = np.random.default_rng(1).permutation(100)
    p = gpu_decode(cv, ctx, code, llr[perm], synd[perm])
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    for x, y in zip(a, sub):
        assert np.array_equal(x[37:90], y)
    for x, y in zip(a, p):
        assert np.array_equal(x[perm], y)


def test_decode_edge_cases(cv, ctx):
    code = codes.regular(96, 3, 6, seed=4)
    u, llr, synd = _channel(code, 33, 2.0, seed=9)
    # max_iter = 0: decision of L only, D = 0 for satisfied frames
    b, cg, it = gpu_decode(cv, ctx, code, llr, synd, max_iter=0)
    b_ref, c_ref, i_ref = oracle.bp_decode(code, llr.astype(np.float64), synd, 0)
    assert np.array_equal(b, b_ref) and np.array_equal(cg, c_ref) and np.array_equal(it, i_ref)
    # noiseless: D = 0 everywhere
    L0 = (40.0 * (1 - 2.0 * u)).astype(np.float32)
    b, cg, it = gpu_decode(cv, ctx, code, L0, synd)
    assert cg.all() and not it.any() and np.array_equal(_brute.unpack_bits(b, code.n), u)
    # frames = 0 is a no-op
    h = load(cv, ctx, code)
    cv.cvsr_decode(ctx, h, None, None, 0, cv.decode_opts(), None, None, None)
    # validation errors
    with pytest.raises(cv.CvsrError) as ei:
        cv.cvsr_decode(ctx, h, None, None, 1, cv.decode_opts(), None, None, None)
    assert ei.value.status == cv.CVSR_EINVAL
    cv.cvsr_code_free(h)
    with pytest.raises(cv.CvsrError) as ei:
        cv.cvsr_code_load(ctx, 4, 1, np.array([0, 2], np.int32), np.array([1, 1], np.int32))
    assert ei.value.status == cv.CVSR_ECODE
    bad = cv.make_quantiser(np.array([0.0, -1.0, 1.0], np.float32))
    with pytest.raises(cv.CvsrError) as ei:
        cv.cvsr_quantise(ctx, bad, 0, 1, 0)
    assert ei.value.status == cv.CVSR_EINVAL


# ------------------------------------------------------------------ reconcile

def _run_reconcile(cv, cfg, codes_l, x, y, F, n, max_iter=100, schedule="default"):
    from paper_2108_08418_b200.pipeline import SRPipeline
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, n, F, torch.device("cuda:0"),
                      max_iter=max_iter, schedule=schedule)
    stats_ = pipe.step(dev(x), dev(y), want_stats=True)
    torch.cuda.synchronize()
    out = dict(label=pipe.label_alice.cpu().numpy(), ok=pipe.frame_ok.cpu().numpy(), iters=pipe.iters.cpu().numpy(),
               bob=pipe.label_bob.cpu().numpy(), synd=[host_u32(s) for s in pipe.synd], stats=stats_,
               errors=pipe.count_errors())
    pipe.close()
    return out


def test_reconcile_parity_c2_scaled(cv, ctx):
    cfg = configs.scaled(configs.C2, 8192, 40)
    codes_l = cfg.build_codes()
    x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=11)
    g = _run_reconcile(cv, cfg, codes_l, x, y, cfg.frames, cfg.n, cfg.max_iter)
    lab_bob = oracle.quantise(cfg.edges(), y)
    assert np.array_equal(g["bob"], lab_bob)
    synd_ref = [oracle.slice_bits(lab_bob, j) if c is None else oracle.syndrome(c, lab_bob, j)
                for j, c in enumerate(codes_l)]
    for s_g, s_r in zip(g["synd"], synd_ref):
        assert np.array_equal(s_g, s_r)
    lab_ref, ok_ref, it_ref = oracle.reconcile(codes_l, cfg.order, cfg.edges(), cfg.sigma_n, x, synd_ref, cfg.max_iter)
    both = ok_ref.astype(bool) & g["ok"].astype(bool)
    assert np.array_equal(g["label"][both], lab_ref[both])
    assert np.sum(g["ok"] != ok_ref) <= max(2, cfg.frames // 20)
    assert np.sum(np.any(g["iters"][both] != it_ref[both], axis=1)) <= max(2, cfg.frames // 20)
    st = g["stats"]
    assert st["frames_ok"] == int(g["ok"].sum())
    assert g["errors"][0] == st["frames_ok"]


def test_reconcile_full_size_sampled(cv, ctx):
    """C2 at full size (n = 2^16) in the bench launch configuration (2048 frames);
    oracle on a sample of frames; properties on all frames."""
    cfg = configs.C2
    codes_l = cfg.build_codes()
    F, n = cfg.frames, cfg.n
    from cvsr_inputs.awgn import torch_quadratures
    xd, yd = torch_quadratures(F, n, cfg.gamma, torch.device("cuda:0"))
    from paper_2108_08418_b200.pipeline import SRPipeline
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, n, F, torch.device("cuda:0"),
                      max_iter=cfg.max_iter)
    st = pipe.step(xd, yd, want_stats=True)
    torch.cuda.synchronize()
    ok = pipe.frame_ok.cpu().numpy()
    assert st["frames_ok"] == int(ok.sum()) and st["frames"] == F
    # every ok frame: Alice's labels reproduce Bob's syndromes exactly (converged => H xhat = s)
    lab_a = pipe.label_alice
    for j, c in enumerate(codes_l):
        if c is None:
            continue
        s_a = torch.empty_like(pipe.synd[j])
        cv.cvsr_syndrome(pipe.ctx, pipe.code_h[j], lab_a, F, j, s_a)
        torch.cuda.synchronize()
        eq = (s_a == pipe.synd[j]).all(dim=1).cpu().numpy()
        assert eq[ok.astype(bool)].all()
    # oracle on sampled frames
    sample = np.array([0, 1, 777, F - 1])
    x = xd[sample].cpu().numpy()
    lab_bob = pipe.label_bob[sample].cpu().numpy()
    synd = [host_u32(s[sample]) for s in pipe.synd]
    lab_ref, ok_ref, it_ref = oracle.reconcile(codes_l, cfg.order, cfg.edges(), cfg.sigma_n, x, synd, cfg.max_iter)
    lab_g = pipe.label_alice[sample].cpu().numpy()
    ok_g = ok[sample]
    both = ok_ref.astype(bool) & ok_g.astype(bool)
    assert np.array_equal(lab_g[both], lab_ref[both])
    assert np.sum(ok_g != ok_ref) <= 1
    assert np.array_equal(lab_ref[ok_ref.astype(bool)], lab_bob[ok_ref.astype(bool)])
    pipe.close()


@pytest.mark.parametrize("name,n,frames", [("C4", 20000, 12), ("C4", 20000, 70), ("C3", 10000, 40)])
def test_reconcile_parity_other_configs(cv, ctx, name, n, frames):
    """C4's 5-slice structure (MET + two irregular codes, incl. a check degree > 8 path) and
    C3's single MET slice, scaled down; 12 frames exercises 1-frame-per-lane tiles (S = 1),
    40/70 frames S = 2 / 4."""
    cfg = configs.scaled(configs.CONFIGS[name], n, frames)
    if name == "C3":
        import dataclasses
        cfg = dataclasses.replace(cfg, gamma=0.2, max_iter=200)  # decodable at n = 1e4
    codes_l = cfg.build_codes()
    x, y = awgn.quadratures(frames, n, cfg.gamma, seed=23)
    g = _run_reconcile(cv, cfg, codes_l, x, y, frames, n, cfg.max_iter)
    lab_bob = oracle.quantise(cfg.edges(), y)
    assert np.array_equal(g["bob"], lab_bob)
    synd_ref = [oracle.slice_bits(lab_bob, j) if c is None else oracle.syndrome(c, lab_bob, j)
                for j, c in enumerate(codes_l)]
    for s_g, s_r in zip(g["synd"], synd_ref):
        assert np.array_equal(s_g, s_r)
    lab_ref, ok_ref, it_ref = oracle.reconcile(codes_l, cfg.order, cfg.edges(), cfg.sigma_n, x, synd_ref,
                                               cfg.max_iter)
    both = ok_ref.astype(bool) & g["ok"].astype(bool)
    assert both.sum() >= 1
    assert np.array_equal(g["label"][both], lab_ref[both])
    assert np.sum(g["ok"] != ok_ref) <= max(1, frames // 20)


@pytest.mark.parametrize("n,frames", [(4096, 40), (2048, 520)])
def test_session_host_and_device_match_pipeline(cv, ctx, n, frames):
    """cvsr_session_run / cvsr_session_run_host (chunked when frames >= 512) reproduce the
    composed pipeline exactly."""
    cfg = configs.scaled(configs.C2, n, frames)
    codes_l = cfg.build_codes()
    x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=41)
    g = _run_reconcile(cv, cfg, codes_l, x, y, cfg.frames, cfg.n, cfg.max_iter)
    hs = [load(cv, ctx, c) if c is not None else None for c in codes_l]
    sess = cv.cvsr_session_create(ctx, cfg.m, hs, cfg.order, cv.make_quantiser(cfg.edges()), cfg.sigma_n, cfg.n,
                                  cfg.frames, cv.decode_opts(cfg.max_iter, 40.0))
    lab = np.empty((cfg.frames, cfg.n), np.uint8)
    ok = np.empty(cfg.frames, np.uint8)
    it = np.empty((cfg.frames, cfg.m), np.int32)
    st = cv.cvsr_session_run_host(sess, np.ascontiguousarray(x), np.ascontiguousarray(y), lab, ok, it,
                                  want_stats=True, m=cfg.m)
    assert np.array_equal(lab, g["label"]) and np.array_equal(ok, g["ok"]) and np.array_equal(it, g["iters"])
    assert st["frames_ok"] == int(ok.sum())
    xd, yd = dev(x), dev(y)
    st2 = cv.cvsr_session_run(sess, xd, yd, want_stats=True, m=cfg.m)
    assert st2["frames_ok"] == st["frames_ok"] and st2["iters_sum"] == st["iters_sum"]
    bob, alice, okp, itp = cv.cvsr_session_buffers(sess)
    assert cv.cvsr_count_errors(ctx, alice, bob, okp, cfg.frames, cfg.n) == g["errors"]
    cv.cvsr_session_destroy(sess)
    for h in hs:
        if h:
            cv.cvsr_code_free(h)


def test_fused_scheduler_subprocess():
    """The experimental fused iteration scheduler (CVSR_FUSED=1) passes the smoke parity check."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CVSR_FUSED="1")
    res = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "smoke OK" in res.stdout


def test_decode_many_frames_compaction_invariance(cv, ctx):
    """600 frames (5 tiles): late iterations compact the active frames into fewer tiles;
    per-frame results must equal decoding each 100-frame slice separately (1 tile, no
    compaction) and, on oracle-converged frames, the oracle."""
    code = codes.regular(1024, 3, 6, seed=1)
    u, llr, synd = _channel(code, 600, 1.5, seed=21)
    full = gpu_decode(cv, ctx, code, llr, synd)
    for a in range(0, 600, 100):
        part = gpu_decode(cv, ctx, code, llr[a:a + 100], synd[a:a + 100])
        for x, y in zip(full, part):
            assert np.array_equal(x[a:a + 100], y)
    b_ref, c_ref, i_ref = oracle.bp_decode(code, llr[:200].astype(np.float64), synd[:200])
    ok = c_ref.astype(bool)
    assert np.array_equal(full[0][:200][ok], b_ref[ok])


def test_compaction_switch_subprocess():
    """CVSR_COMPACT=0 and =1 give bit-identical reconcile results (C2 structure, 520 frames)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = (
        "import numpy as np, torch\n"
        "from cvsr_inputs import awgn, configs\n"
        "from paper_2108_08418_b200.pipeline import SRPipeline\n"
        "cfg = configs.scaled(configs.C2, 2048, 520)\n"
        "cl = cfg.build_codes()\n"
        "x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=5)\n"
        "p = SRPipeline(cfg.m, cfg.edges(), cl, cfg.order, cfg.sigma_n, cfg.n, cfg.frames, torch.device('cuda:0'))\n"
        "p.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())\n"
        "torch.cuda.synchronize()\n"
        "np.save(__import__('sys').argv[1], np.concatenate([p.label_alice.cpu().numpy().ravel(),"
        " p.iters.cpu().numpy().ravel().astype(np.uint8), p.frame_ok.cpu().numpy()]))\n")
    import tempfile
    outs = []
    for flag in ("0", "1"):
        f = tempfile.mktemp(suffix=".npy")
        res = subprocess.run([sys.executable, "-c", prog, f], cwd=root, env=dict(os.environ, CVSR_COMPACT=flag),
                             capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


# ----------------------------------------------------------------- verification hash (R-6)
@pytest.mark.parametrize("n", [1, 3, 5, 255, 1024, 4097, 65536, 262147])
def test_frame_hash_and_verify_bitexact(cv, ctx, n):
    """cvsr_frame_hash / cvsr_verify equal the oracle's polynomial hash bit for bit (aligned and
    ragged n; n = 262147 takes the 1024-thread blocks used for few long frames); verified =
    frame_ok AND equal hashes; a single flipped label bit is caught."""
    from oracle import verify
    rng = np.random.default_rng(n)
    F = 6 if n < 65536 else 3
    lab_b = rng.integers(0, 32, size=(F, n), dtype=np.uint8)
    lab_a = lab_b.copy()
    lab_a[1, rng.integers(0, n)] ^= np.uint8(1 << rng.integers(0, 5))       # frame 1 wrong
    ok = np.ones(F, np.uint8)
    ok[2] = 0                                                               # frame 2 not converged
    da, db, dok = dev(lab_a), dev(lab_b), dev(ok)
    key_list = (1, 1 << 32, int(rng.integers(1, verify.P61 - 1)), verify.P61 - 2)
    for key in key_list:
        h = torch.empty(F, dtype=torch.int64, device="cuda")
        cv.cvsr_frame_hash(ctx, da, F, n, key, h)
        assert np.array_equal(h.cpu().numpy().astype(np.uint64), verify.frame_hash(lab_a, key))
    for keys in (key_list[:3], key_list[1:]):
        ha = torch.empty((F, cv.CVSR_HASH_KEYS), dtype=torch.int64, device="cuda")
        hb = torch.empty_like(ha)
        ver = torch.empty(F, dtype=torch.uint8, device="cuda")
        cv.cvsr_verify(ctx, da, db, dok, F, n, keys, ver, ha, hb)
        for q, key in enumerate(keys):
            assert np.array_equal(ha[:, q].cpu().numpy().astype(np.uint64), verify.frame_hash(lab_a, key))
            assert np.array_equal(hb[:, q].cpu().numpy().astype(np.uint64), verify.frame_hash(lab_b, key))
        want = ok.copy()
        want[1] = 0
        assert np.array_equal(ver.cpu().numpy(), want)
    with pytest.raises(cv.CvsrError):
        cv.cvsr_verify(ctx, da, db, dok, F, n, (1, 0, 2), ver, ha, hb)
    with pytest.raises(cv.CvsrError):
        cv.cvsr_frame_hash(ctx, da, F, n, 0, h)
    cv.cvsr_frame_hash(ctx, da, 0, n, 5, h)   # empty batch is a no-op


def test_reconcile_then_verify(cv, ctx):
    """After reconciliation the hash check passes exactly on the frames whose labels equal Bob's
    (the session's in-place variant agrees)."""
    cfg = configs.scaled(configs.C2, 4096, 48)
    codes_l = cfg.build_codes()
    x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=5)
    from paper_2108_08418_b200.pipeline import SRPipeline
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, cfg.frames, torch.device("cuda:0"),
                      max_iter=cfg.max_iter)
    pipe.step(dev(x), dev(y), key=(0x1234567, 0x7654321, 0xABCDEF))
    torch.cuda.synchronize()
    same = (pipe.label_alice == pipe.label_bob).all(dim=1).cpu().numpy()
    ok = pipe.frame_ok.cpu().numpy().astype(bool)
    assert np.array_equal(pipe.verified.cpu().numpy().astype(bool), ok & same)
    hs = [load(cv, ctx, c) if c is not None else None for c in codes_l]
    sess = cv.cvsr_session_create(ctx, cfg.m, hs, cfg.order, cv.make_quantiser(cfg.edges()), cfg.sigma_n, cfg.n,
                                  cfg.frames, cv.decode_opts(cfg.max_iter, 40.0))
    cv.cvsr_session_set_verify(sess, (0x1234567, 0x7654321, 0xABCDEF))
    lab = np.empty((cfg.frames, cfg.n), np.uint8)
    okh = np.empty(cfg.frames, np.uint8)
    it = np.empty((cfg.frames, cfg.m), np.int32)
    cv.cvsr_session_run_host(sess, np.ascontiguousarray(x), np.ascontiguousarray(y), lab, okh, it)
    assert np.array_equal(okh, pipe.verified.cpu().numpy())
    cv.cvsr_session_destroy(sess)
    for h in hs:
        if h:
            cv.cvsr_code_free(h)
    pipe.close()


@pytest.mark.parametrize("n,frames", [(4096, 40), (2048, 520)])
def test_session_stream_matches_run_host(cv, ctx, n, frames):
    """cvsr_session_run_host_stream (double-buffered batches) returns, per batch, exactly what
    cvsr_session_run_host (which chunks batches of >= 512 frames) returns for that batch alone
    (3 batches, hash check on)."""
    cfg = configs.scaled(configs.C2, n, frames)
    codes_l = cfg.build_codes()
    hs = [load(cv, ctx, c) if c is not None else None for c in codes_l]
    sess = cv.cvsr_session_create(ctx, cfg.m, hs, cfg.order, cv.make_quantiser(cfg.edges()), cfg.sigma_n, cfg.n,
                                  cfg.frames, cv.decode_opts(cfg.max_iter, 40.0))
    cv.cvsr_session_set_verify(sess, (987654321, 123456789, 555555555))
    xs, ys, want_lab, want_ok = [], [], [], []
    for b in range(3):
        x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=100 + b)
        x, y = np.ascontiguousarray(x), np.ascontiguousarray(y)
        lab = np.empty((cfg.frames, cfg.n), np.uint8)
        ok = np.empty(cfg.frames, np.uint8)
        cv.cvsr_session_run_host(sess, x, y, lab, ok)
        xs.append(x), ys.append(y), want_lab.append(lab), want_ok.append(ok)
    labs = [np.full((cfg.frames, cfg.n), 255, np.uint8) for _ in range(3)]
    oks = [np.full(cfg.frames, 255, np.uint8) for _ in range(3)]
    cv.cvsr_session_run_host_stream(sess, xs, ys, labs, oks)
    for b in range(3):
        assert np.array_equal(labs[b], want_lab[b]) and np.array_equal(oks[b], want_ok[b])
    # labels may be skipped; a second call reuses the buffer sets
    oks2 = [np.zeros(cfg.frames, np.uint8) for _ in range(3)]
    cv.cvsr_session_run_host_stream(sess, xs, ys, [None, None, None], oks2)
    assert all(np.array_equal(a, b) for a, b in zip(oks2, want_ok))
    cv.cvsr_session_destroy(sess)
    for h in hs:
        if h:
            cv.cvsr_code_free(h)


# ----------------------------------------------------------------- Toeplitz privacy amplification (R-8)
@pytest.mark.parametrize("n_in,n_out,blocks,sample", [(1, 1, 2, None), (5, 3, 3, None), (100, 37, 2, None),
                                                      (2048, 2048, 2, None), (4097, 4096, 1, None),
                                                      (4096, 1000, 2, None), (5000, 4999, 1, None),
                                                      (20000, 7000, 3, None), (1 << 16, 1 << 15, 2, 300),
                                                      ((1 << 20) + 3, 777_777, 1, 64)])
def test_pa_toeplitz_bitexact(cv, ctx, n_in, n_out, blocks, sample):
    """cvsr_pa_hash equals the oracle's row-by-row Toeplitz product bit for bit (all rows, or
    `sample` random rows at the larger sizes); sizes cover N = 2 .. 2^21 (shared-memory-only
    transforms and 1-4-stage global passes), n_in = n_out, N exactly 4096 (shared-memory
    kernel only) and n_in + n_out - 1 = 2^13 exactly, and ragged bit counts."""
    from oracle import pa
    rng = np.random.default_rng(n_in + n_out)
    t = rng.integers(0, 2, n_in + n_out - 1, dtype=np.uint8)
    plan = cv.cvsr_pa_plan_create(ctx, n_in, n_out, pa.pack_bits(t))
    assert cv.cvsr_pa_plan_info(plan)[:2] == (n_in, n_out)
    xs = [rng.integers(0, 2, n_in, dtype=np.uint8) for _ in range(blocks)]
    xd = dev(np.stack([pa.pack_bits(x) for x in xs]))
    wo = (n_out + 31) // 32
    yd = torch.empty((blocks, wo), dtype=torch.int32, device="cuda")
    cv.cvsr_pa_hash(ctx, plan, blocks, xd, yd)
    yh = host_u32(yd)
    for b in range(blocks):
        got = pa.unpack_bits(yh[b], n_out)
        if sample is None:
            assert np.array_equal(got, pa.toeplitz_hash(t, xs[b], n_out))
            assert (n_out % 32 == 0) or (yh[b][-1] >> (n_out % 32)) == 0
        else:
            rows = np.sort(rng.choice(n_out, size=sample, replace=False))
            rows = np.unique(np.concatenate([rows, [0, n_out - 1]]))
            assert np.array_equal(got[rows], pa.toeplitz_hash(t, xs[b], n_out, rows=rows))
    cv.cvsr_pa_plan_free(plan)


def test_pa_errors(cv, ctx):
    with pytest.raises(cv.CvsrError):
        cv.cvsr_pa_plan_create(ctx, 10, 11, np.zeros(1, np.uint32))     # n_out > n_in
    with pytest.raises(cv.CvsrError):
        cv.cvsr_pa_plan_create(ctx, 1 << 27, 2, np.zeros((1 << 22) + 1, np.uint32))  # > 2^27


def test_sharded_reconcile_equals_single_batch(cv, ctx):
    """what rank r of k computes for its frame range (inputs from the
    shard-invariant generator the bench uses, `first_frame = r F`) equals the same frames of one
    k F-frame run -- labels, flags, iteration counts and hashes -- for k = 2 and 4."""
    from cvsr_inputs.awgn import torch_quadratures
    from paper_2108_08418_b200 import dist as cdist
    from paper_2108_08418_b200.pipeline import SRPipeline
    cfg = configs.scaled(configs.C2, 4096, 64)
    codes_l = cfg.build_codes()
    dev0 = torch.device("cuda:0")
    F = cfg.frames

    def run(frames, first):
        x, y = torch_quadratures(frames, cfg.n, cfg.gamma, dev0, first_frame=first)
        p = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, frames, dev0, max_iter=cfg.max_iter)
        p.step(x, y, key=(12345, 67890, 13579))
        torch.cuda.synchronize()
        out = (p.label_alice.cpu().numpy(), p.verified.cpu().numpy(), p.iters.cpu().numpy(), p.hash_alice.cpu().numpy())
        p.close()
        return out

    for k in (2, 4):
        full = run(k * F, 0)
        for r in range(k):
            first, nloc = cdist.shard(F, r)
            assert nloc == F and first == r * F
            part = run(F, first)
            for a, b in zip(part, full):
                assert np.array_equal(a, b[r * F:(r + 1) * F])


def test_graph_replay_and_smem_decoder_match_launch_loop():
    """Three implementations of the same iterations give identical decoded bits, flags and
    iteration counts on C1: the plain launch loop (CVSR_SMEM=0 CVSR_GRAPH=0), its CUDA-graph
    replay (CVSR_GRAPH=1) and the one-CTA-per-frame shared-memory decoder (CVSR_SMEM=1)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = r'''
import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from cvsr_inputs import awgn, codes
from paper_2108_08418_b200 import cvsr as cv
code = codes.regular(1024, 3, 6, seed=1)
sigma = awgn.biawgn_sigma(0.5, 1.5)
u, y = awgn.biawgn(100, 1024, sigma, seed=77)
ctx = cv.cvsr_ctx_create(0, torch.cuda.current_stream())
h = cv.cvsr_code_load(ctx, code.n, code.m_checks, code.row_ptr, code.col_idx)
lab = torch.from_numpy(u).cuda()
synd = torch.empty((100, 16), dtype=torch.int32, device="cuda")
cv.cvsr_syndrome(ctx, h, lab, 100, 0, synd)
yd = torch.from_numpy(y).cuda(); llr = torch.empty_like(yd)
cv.cvsr_llr_biawgn(ctx, yd, y.size, sigma ** 2, 40.0, llr)
bits = torch.empty((100, 32), dtype=torch.int32, device="cuda")
conv = torch.empty(100, dtype=torch.uint8, device="cuda"); it = torch.empty(100, dtype=torch.int32, device="cuda")
cv.cvsr_decode(ctx, h, llr, synd, 100, cv.decode_opts(100, 40.0), bits, conv, it)
torch.cuda.synchronize()
np.savez(sys.argv[1], bits=bits.cpu().numpy(), conv=conv.cpu().numpy(), it=it.cpu().numpy())
'''
    def run(env, tag):
        path = os.path.join(root, "gpurun_out", f"dec_{tag}.npz") if os.path.isdir(os.path.join(root, "gpurun_out")) \
            else f"/tmp/dec_{tag}.npz"
        res = subprocess.run([sys.executable, "-c", prog, path], cwd=root, env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        return np.load(path)

    # graph replay vs plain launches (interleaved path), and the shared-memory decoder vs both
    outs = [run({"CVSR_SMEM": "0", "CVSR_GRAPH": "1"}, "graph"), run({"CVSR_SMEM": "0", "CVSR_GRAPH": "0"}, "loop"),
            run({"CVSR_SMEM": "1"}, "smem")]
    for o in outs[1:]:
        for k in ("bits", "conv", "it"):
            assert np.array_equal(outs[0][k], o[k]), k
    assert outs[0]["conv"].sum() >= 50


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_smem_decoder_reconcile_matches_interleaved(name):
    """Whole reconciles (several slices, frames that stop after a failed slice, MET codes with
    degree-2 checks) give identical labels, flags and iteration counts with the shared-memory
    decoder (n = 2048 fits its 40 KB limit; the launch count shows it was taken) and with the
    interleaved kernels (CVSR_SMEM=0)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = r'''
import sys, dataclasses, numpy as np, torch
sys.path.insert(0, ".")
from cvsr_inputs import awgn, configs
from paper_2108_08418_b200.pipeline import SRPipeline
cfg = configs.scaled(configs.CONFIGS[sys.argv[2]], 2048, 200)
if sys.argv[2] == "C4":
    cfg = dataclasses.replace(cfg, gamma=2.2)   # n = 2048 at the standard SNR: about 2/3 of the frames fail
codes_l = cfg.build_codes()
x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=31)
p = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, cfg.frames, torch.device("cuda:0"),
               max_iter=cfg.max_iter)
p.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
torch.cuda.synchronize()
np.savez(sys.argv[1], lab=p.label_alice.cpu().numpy(), ok=p.frame_ok.cpu().numpy(), it=p.iters.cpu().numpy(),
         launches=np.array([p.launches()]))
'''
    outs = []
    for flag in ("1", "0"):
        path = os.path.join(root, "gpurun_out", f"rec_{name}_{flag}.npz") \
            if os.path.isdir(os.path.join(root, "gpurun_out")) else f"/tmp/rec_{name}_{flag}.npz"
        res = subprocess.run([sys.executable, "-c", prog, path, name], cwd=root,
                             env=dict(os.environ, CVSR_SMEM=flag), capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(np.load(path))
    for k in ("lab", "ok", "it"):
        assert np.array_equal(outs[0][k], outs[1][k]), k
    assert outs[0]["ok"].sum() >= 1
    assert outs[0]["launches"][0] < outs[1]["launches"][0] // 2   # the on-chip decoder was used


def test_tile_width_and_fused_scheduler_bit_identical():
    """The frames-per-lane choice (CVSR_SUBS = 1, 2, 4) and the experimental fused scheduler
    (CVSR_FUSED=1) change only the schedule: a multi-tile C2-structure reconcile gives identical
    labels, flags and iteration counts."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prog = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from cvsr_inputs import awgn, configs
from paper_2108_08418_b200.pipeline import SRPipeline
cfg = configs.scaled(configs.C2, 8192, 300)
codes_l = cfg.build_codes()
x, y = awgn.quadratures(cfg.frames, cfg.n, cfg.gamma, seed=12)
p = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, cfg.frames, torch.device("cuda:0"),
               max_iter=cfg.max_iter)
p.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
torch.cuda.synchronize()
np.savez(sys.argv[1], lab=p.label_alice.cpu().numpy(), ok=p.frame_ok.cpu().numpy(), it=p.iters.cpu().numpy())
'''
    outs = []
    for tag, env in (("s4", {"CVSR_SUBS": "4"}), ("s2", {"CVSR_SUBS": "2"}), ("s1", {"CVSR_SUBS": "1"}),
                     ("fused", {"CVSR_FUSED": "1"})):
        path = os.path.join(root, "gpurun_out", f"sub_{tag}.npz") if os.path.isdir(os.path.join(root, "gpurun_out")) \
            else f"/tmp/sub_{tag}.npz"
        res = subprocess.run([sys.executable, "-c", prog, path], cwd=root, env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, res.stderr[-2000:]
        outs.append(np.load(path))
    for o in outs[1:]:
        for k in ("lab", "ok", "it"):
            assert np.array_equal(outs[0][k], o[k]), k


# ------------------------------------------------------------------ row-layered schedule (reading R-9)
