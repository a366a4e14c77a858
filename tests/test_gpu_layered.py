"""Row-layered schedule (reading R-9) of the CUDA path vs the oracle's layered
decoder / layered multi-stage driver, through the C ABI with
cvsr_decode_opts.flags = CVSR_SCHED_LAYERED (the bench's launch configuration).

Parity criteria as for flooding: messages r_e and posteriors after
k in {1, 2, 5, 10} iterations within |gpu - ref| <= 1e-4 (|ref| + 1) (reading A-22);
decoded bits identical on every frame where the oracle converges; convergence flags and
iteration counts differ on at most a few percent of frames (fp32 vs fp64 rounding near
a decision); FER inside the oracle's 95 % interval.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import _brute
import oracle
from cvsr_inputs import awgn, codes, configs
from test_gpu_parity import TOL, _channel, _clopper_pearson, _run_reconcile, dev, host_u32, load, rel_err

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cv(gpu):
    from paper_2108_08418_b200 import cvsr
    return cvsr


@pytest.fixture(scope="module")
def ctx(cv):
    c = cv.cvsr_ctx_create(0, torch.cuda.current_stream())
    yield c
    cv.cvsr_ctx_destroy(c)


# codes whose layered kernels the bench configurations use: C1's (3,6) (k_layer<6>), C2's coded
# slices (<5>), C4's S3 (check degrees 8/9: <9>), S4 (6/7: <7>) and MET S2 (degree-2 type-A
# checks + degree-6 core: <6> with the 2-edge body), a small MET code and a ragged n
LAYER_CODES = {
    "c1_36": lambda: codes.regular(1024, 3, 6, seed=1),
    "c2_s2": lambda: codes.irregular_rate(4100, 0.356, seed=3, lam=dict(configs.LAMBDA_C2)),
    "c4_s3": lambda: codes.irregular_rate(20000, 0.583, seed=3),
    "c4_s4": lambda: codes.irregular_rate(20000, 0.442, seed=4),
    "c4_s2_met": lambda: codes.met_low_rate(20000, 0.10, 0.05, 3, 6, seed=5),
    "met_small": lambda: codes.met_low_rate(2000, 0.04, 0.02, 3, 6, seed=5),
}
EBN0 = {"c1_36": 1.5, "c2_s2": 1.0, "c4_s3": 2.0, "c4_s4": 1.5, "c4_s2_met": -1.0, "met_small": -1.0}

LAYERED = 2  # CVSR_SCHED_LAYERED
FLOODING = 1


def gpu_decode(cv, ctx, code, llr32, synd, max_iter=100, flags=LAYERED):
    F = llr32.shape[0]
    h = load(cv, ctx, code)
    bits = torch.empty((F, (code.n + 31) // 32), dtype=torch.int32, device="cuda")
    conv = torch.empty(F, dtype=torch.uint8, device="cuda")
    iters = torch.empty(F, dtype=torch.int32, device="cuda")
    cv.cvsr_decode(ctx, h, dev(llr32), dev(synd), F, cv.decode_opts(max_iter, 40.0, flags), bits, conv, iters)
    cv.cvsr_ctx_sync(ctx)
    cv.cvsr_code_free(h)
    return host_u32(bits), conv.cpu().numpy(), iters.cpu().numpy()


def gpu_trace(cv, ctx, code, llr32, synd, k):
    F = llr32.shape[0]
    h = load(cv, ctx, code)
    r = torch.empty((F, code.n_edges), dtype=torch.float32, device="cuda")
    post = torch.empty((F, code.n), dtype=torch.float32, device="cuda")
    cv.cvsr_decode_trace(ctx, h, dev(llr32), dev(synd), F, k, 40.0, r, post, flags=LAYERED)
    cv.cvsr_ctx_sync(ctx)
    cv.cvsr_code_free(h)
    return r.cpu().numpy(), post.cpu().numpy()


@pytest.mark.parametrize("name,F", [(k, 45) for k in LAYER_CODES] + [("c4_s3", 12), ("c2_s2", 12)])
def test_layered_trace_messages_parity(cv, ctx, name, F):
    """r_e (CSR order) and posteriors after exactly k layered iterations vs the oracle's layered
    trace (PAPER.md:189 BP, PAPER.md:231 per-iteration messages): 45 frames = two 32-frame
    tiles or one ragged 64-frame tile; 12 frames = one ragged tile."""
    code = LAYER_CODES[name]()
    u, llr, synd = _channel(code, F, EBN0[name], seed=7)
    for k in (1, 2, 5, 10):
        r_ref, post_ref = oracle.bp_trace_layered(code, llr.astype(np.float64), synd, k)
        r, post = gpu_trace(cv, ctx, code, llr, synd, k)
        assert rel_err(r, r_ref) <= TOL, (k, rel_err(r, r_ref))
        assert rel_err(post, post_ref) <= TOL, (k, rel_err(post, post_ref))


def test_layered_tree_exact_marginals_gpu(cv, ctx):
    """Cycle-free Tanner graphs: the layered CUDA decoder reaches the exact MAP marginals."""
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


def _layered_cases():
    """(name, code, F, E_b/N_0, seed, max_iter): C1, C2's coded-slice ensemble (ragged 200 frames;
    600 frames for compaction), C4's slice codes, one frame, max_iter = 0."""
    c1 = codes.regular(1024, 3, 6, seed=configs.CODE_SEED)
    return [("c1", c1, 100, 1.5, 1, 100),
            ("c2s2", codes.irregular_rate(4096, 0.356, seed=3, lam=dict(configs.LAMBDA_C2)), 200, 1.0, 2, 100),
            ("c2s3", codes.irregular_rate(2048, 0.257, seed=4, lam=dict(configs.LAMBDA_C2)), 600, 1.5, 3, 100),
            ("c4s3", LAYER_CODES["c4_s3"](), 70, 2.2, 6, 100),
            ("c4s4", LAYER_CODES["c4_s4"](), 40, 1.6, 8, 100),
            ("c4met", LAYER_CODES["c4_s2_met"](), 70, -0.5, 9, 100),
            ("one", c1, 1, 2.0, 4, 100), ("zero", c1, 40, 1.5, 5, 0)]


@pytest.mark.parametrize("case", _layered_cases(), ids=lambda c: c[0])
def test_layered_decode_parity(cv, ctx, case):
    """cvsr_decode with CVSR_SCHED_LAYERED vs the oracle's row-layered decoder: decisions identical
    on every frame where the oracle converges, at most 2 % of frames with a different D or flag,
    FER inside the oracle's 95 % interval, converged => H xhat = s, and fewer mean iterations than
    the flooding oracle on the same frames."""
    name, code, F, ebn0, seed, mi = case
    u, llr, synd = _channel(code, F, ebn0, seed)
    b, cg, it = gpu_decode(cv, ctx, code, llr, synd, mi)
    b_ref, c_ref, i_ref, _ = oracle.bp_decode_layered(code, llr.astype(np.float64), synd, mi)
    ok = c_ref.astype(bool)
    assert np.array_equal(b[ok & (cg == 1)], b_ref[ok & (cg == 1)]), name
    assert np.sum(cg != c_ref) <= max(1, F // 50), (name, int(np.sum(cg != c_ref)))
    assert np.sum(it != i_ref) <= max(1, F // 50), (name, int(np.sum(it != i_ref)))
    lo, hi = _clopper_pearson(int(np.sum(c_ref == 0)), F)
    assert lo <= float(np.mean(cg == 0)) <= hi, name
    s_dec = oracle.syndrome(code, _brute.unpack_bits(b, code.n), 0)
    for f in range(F):
        if cg[f]:
            assert np.array_equal(s_dec[f], synd[f]), (name, f)
    if name in ("c1", "c2s2", "c2s3", "c4s3", "c4s4"):
        _, cf, df = oracle.bp_decode(code, llr.astype(np.float64), synd, mi)
        both = (cf == 1) & (cg == 1)
        assert both.sum() >= F // 2 and it[both].mean() < 0.8 * df[both].mean(), name


def test_layered_env_default_matches_flag(cv, tmp_path):
    """CVSR_SCHEDULE=layered makes CVSR_SCHED_DEFAULT run the layered schedule: bit-identical to
    an explicit CVSR_SCHED_LAYERED (subprocess: the variable is read once per process)."""
    code = codes.irregular_rate(4096, 0.356, seed=3, lam=dict(configs.LAMBDA_C2))
    u, llr, synd = _channel(code, 100, 1.0, 2)
    np.savez(tmp_path / "in.npz", rp=code.row_ptr, ci=code.col_idx, llr=llr, synd=synd,
             dims=np.array([code.n, code.m_checks]))
    child = (
        "import sys, numpy as np, torch\n"
        "from paper_2108_08418_b200 import cvsr as cv\n"
        "d = np.load(sys.argv[1]); n, M = (int(v) for v in d['dims']); F = d['llr'].shape[0]\n"
        "ctx = cv.cvsr_ctx_create(0, torch.cuda.current_stream())\n"
        "h = cv.cvsr_code_load(ctx, n, M, d['rp'], d['ci'])\n"
        "out = {}\n"
        "for tag, fl in (('dflt', 0), ('lay', 2), ('flood', 1)):\n"
        "    b = torch.empty((F, (n + 31) // 32), dtype=torch.int32, device='cuda')\n"
        "    c = torch.empty(F, dtype=torch.uint8, device='cuda'); it = torch.empty(F, dtype=torch.int32, device='cuda')\n"
        "    cv.cvsr_decode(ctx, h, torch.from_numpy(d['llr']).cuda(), torch.from_numpy(d['synd'].view(np.int32)).cuda(),\n"
        "                   F, cv.decode_opts(100, 40.0, fl), b, c, it)\n"
        "    cv.cvsr_ctx_sync(ctx)\n"
        "    out[tag + '_b'] = b.cpu().numpy(); out[tag + '_i'] = it.cpu().numpy()\n"
        "np.savez(sys.argv[2], **out)\n")
    res = subprocess.run([sys.executable, "-c", child, str(tmp_path / "in.npz"), str(tmp_path / "out.npz")], cwd=ROOT,
                         env=dict(os.environ, CVSR_SCHEDULE="layered",
                                  PYTHONPATH=os.pathsep.join([ROOT, os.environ.get("PYTHONPATH", "")])),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    o = np.load(tmp_path / "out.npz")
    assert np.array_equal(o["dflt_b"], o["lay_b"]) and np.array_equal(o["dflt_i"], o["lay_i"])
    assert o["flood_i"].mean() > o["lay_i"].mean()


def test_layered_unsupported_code_falls_back_to_flooding(cv, ctx):
    """A check degree > 12 has no layered kernel: CVSR_SCHED_LAYERED decodes that code with
    flooding (bit-identical to CVSR_SCHED_FLOODING) instead of failing the call, and
    cvsr_reconcile reports the schedule that ran per slice; the layered trace is refused."""
    code = codes.regular(1500, 3, 15, seed=2)
    u, llr, synd = _channel(code, 37, 2.5, 3)
    a = gpu_decode(cv, ctx, code, llr, synd, flags=LAYERED)
    b = gpu_decode(cv, ctx, code, llr, synd, flags=FLOODING)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    h = load(cv, ctx, code)
    with pytest.raises(cv.CvsrError) as ei:
        cv.cvsr_decode_trace(ctx, h, dev(llr), dev(synd), 37, 2, 40.0, None, None, flags=LAYERED)
    assert ei.value.status == cv.CVSR_EINVAL
    with pytest.raises(cv.CvsrError):
        cv.cvsr_decode(ctx, h, dev(llr), dev(synd), 37, cv.decode_opts(10, 40.0, 3), None, None, None)
    cv.cvsr_code_free(h)
    # reconcile: m = 1 sign slice with that code
    import dataclasses
    cfg = dataclasses.replace(configs.scaled(configs.C3, 1500, 37), gamma=8.0, max_iter=100)
    x, y = awgn.quadratures(37, 1500, cfg.gamma, seed=5)
    g = _run_reconcile(cv, cfg, [code], x, y, 37, 1500, 100, schedule="layered")
    assert g["stats"]["schedule"] == [FLOODING]
    g2 = _run_reconcile(cv, cfg, [codes.regular(1500, 3, 6, seed=2)], x, y, 37, 1500, 100, schedule="layered")
    assert g2["stats"]["schedule"] == [LAYERED]


def _reconcile_case(name, n, frames):
    cfg = configs.scaled(configs.CONFIGS[name], n, frames)
    if name == "C3":
        import dataclasses
        cfg = dataclasses.replace(cfg, gamma=0.2, max_iter=200)  # decodable at n = 1e4
    return cfg


@pytest.mark.parametrize("name,n,frames", [("C2", 8192, 40), ("C2", 4096, 130), ("C4", 20000, 12),
                                           ("C4", 20000, 70), ("C3", 10000, 40)])
def test_reconcile_layered_parity(cv, ctx, name, n, frames):
    """cvsr_reconcile under CVSR_SCHED_LAYERED (the bench's schedule) vs the oracle's layered
    multi-stage driver O6 (PAPER.md:114 steps 4-6): Bob's labels and syndromes bit-exact;
    Alice's labels identical on every frame both sides reconcile; flags and per-slice D differ
    on at most 5 % of frames; every slice ran layered.  C4's slices exercise k_layer<6> with
    the degree-2 body (MET S2), <9> (S3) and <7> (S4) at one frame per lane."""
    cfg = _reconcile_case(name, n, frames)
    codes_l = cfg.build_codes()
    x, y = awgn.quadratures(frames, n, cfg.gamma, seed=23)
    g = _run_reconcile(cv, cfg, codes_l, x, y, frames, n, cfg.max_iter, schedule="layered")
    lab_bob = oracle.quantise(cfg.edges(), y)
    assert np.array_equal(g["bob"], lab_bob)
    synd_ref = [oracle.slice_bits(lab_bob, j) if c is None else oracle.syndrome(c, lab_bob, j)
                for j, c in enumerate(codes_l)]
    for s_g, s_r in zip(g["synd"], synd_ref):
        assert np.array_equal(s_g, s_r)
    lab_ref, ok_ref, it_ref = oracle.reconcile(codes_l, cfg.order, cfg.edges(), cfg.sigma_n, x, synd_ref,
                                               cfg.max_iter, schedule="layered")
    both = ok_ref.astype(bool) & g["ok"].astype(bool)
    assert both.sum() >= max(1, frames // 2)
    assert np.array_equal(g["label"][both], lab_ref[both])
    # a converged frame can still be a wrong codeword at these short lengths (the MET code's
    # low-weight codewords); both implementations then agree on it (above) and the hash check
    # discards it -- the full-size C4 test below requires none at N_R = 1e6
    okr = ok_ref.astype(bool)
    assert np.sum(np.any(lab_ref[okr] != lab_bob[okr], axis=1)) <= max(1, frames // 50)
    assert np.sum(g["ok"] != ok_ref) <= max(1, frames // 20)
    assert np.sum(np.any(g["iters"][both] != it_ref[both], axis=1)) <= max(1, frames // 20)
    st = g["stats"]
    assert st["schedule"] == [0 if c is None else LAYERED for c in codes_l]
    assert st["frames_ok"] == int(g["ok"].sum()) and g["errors"][0] == st["frames_ok"]


def test_reconcile_layered_c4_full_size_sampled(cv, ctx):
    """C4 at full size (N_R = 10^6, 125 frames: the bench's launch configuration and schedule):
    every reconciled frame reproduces Bob's syndromes of every coded slice; the oracle's layered
    driver on two sampled frames agrees label for label."""
    cfg = configs.C4
    codes_l = cfg.build_codes()
    F, n = cfg.frames, cfg.n
    from cvsr_inputs.awgn import torch_quadratures
    from paper_2108_08418_b200.pipeline import SRPipeline
    xd, yd = torch_quadratures(F, n, cfg.gamma, torch.device("cuda:0"))
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, n, F, torch.device("cuda:0"),
                      max_iter=cfg.max_iter, schedule="layered")
    st = pipe.step(xd, yd, want_stats=True)
    torch.cuda.synchronize()
    ok = pipe.frame_ok.cpu().numpy().astype(bool)
    assert st["frames"] == F and st["frames_ok"] == int(ok.sum()) and ok.mean() > 0.9
    assert st["schedule"] == [0 if c is None else LAYERED for c in codes_l]
    for j, c in enumerate(codes_l):
        if c is None:
            continue
        s_a = torch.empty_like(pipe.synd[j])
        cv.cvsr_syndrome(pipe.ctx, pipe.code_h[j], pipe.label_alice, F, j, s_a)
        torch.cuda.synchronize()
        assert (s_a == pipe.synd[j]).all(dim=1).cpu().numpy()[ok].all()
    assert pipe.count_errors()[1] == 0
    sample = np.array([0, F - 1])
    x = xd[sample].cpu().numpy()
    synd = [host_u32(s[sample]) for s in pipe.synd]
    lab_ref, ok_ref, it_ref = oracle.reconcile(codes_l, cfg.order, cfg.edges(), cfg.sigma_n, x, synd, cfg.max_iter,
                                               schedule="layered")
    lab_g = pipe.label_alice[sample].cpu().numpy()
    both = ok_ref.astype(bool) & ok[sample]
    assert both.sum() >= 1 and np.array_equal(lab_g[both], lab_ref[both])
    pipe.close()


def test_layered_variants_bit_identical(tmp_path):
    """Every layered kernel variant performs the same arithmetic in the same layer order, so the
    frames-per-lane choice (CVSR_SUBS = 1, 2, 4), the register-staged k_layer (CVSR_LAYER_TMA=0),
    the persistent k_layer_tmap (CVSR_LAYER_PERSIST=1), frame compaction off (CVSR_COMPACT=0),
    plain stream-ordered layer launches (CVSR_LAYER_PDL=0), no reads before the dependency wait
    (CVSR_LAYER_EARLY=0), the thread-per-(check, tile) syndrome test (CVSR_SYND_TEST_W=0) and
    Bob's per-frame syndrome kernels (CVSR_SYND_SLICED=0), degree <= 2 checks in 4-check chunks
    (CVSR_LAYER_PAIRS=0) or always in 12-check chunks (CVSR_LAYER_CH2_WAVES=0; at these sizes the
    default takes 4) give bit-identical labels, flags and iteration counts on a multi-tile C4-structure and C2
    reconcile."""
    prog = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from cvsr_inputs import awgn, configs
from paper_2108_08418_b200.pipeline import SRPipeline
out = {}
for name, n, F in (("C4", 20000, 150), ("C2", 8192, 200)):
    cfg = configs.scaled(configs.CONFIGS[name], n, F)
    codes_l = cfg.build_codes()
    x, y = awgn.quadratures(F, n, cfg.gamma, seed=44)
    p = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, n, F, torch.device("cuda:0"),
                   max_iter=cfg.max_iter, schedule="layered")
    p.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    torch.cuda.synchronize()
    out[name + "_lab"] = p.label_alice.cpu().numpy()
    out[name + "_ok"] = p.frame_ok.cpu().numpy()
    out[name + "_it"] = p.iters.cpu().numpy()
    p.close()
np.savez(sys.argv[1], **out)
'''
    outs = []
    for tag, env in (("default", {}), ("s1", {"CVSR_SUBS": "1"}), ("s4", {"CVSR_SUBS": "4"}),
                     ("reg", {"CVSR_LAYER_TMA": "0"}), ("persist", {"CVSR_LAYER_PERSIST": "1"}),
                     ("nocompact", {"CVSR_COMPACT": "0"}), ("nopdl", {"CVSR_LAYER_PDL": "0"}),
                     ("noearly", {"CVSR_LAYER_EARLY": "0"}), ("synd_test_thread", {"CVSR_SYND_TEST_W": "0"}),
                     ("bob_synd_per_frame", {"CVSR_SYND_SLICED": "0"}), ("nopairs", {"CVSR_LAYER_PAIRS": "0"}),
                     ("pairs12", {"CVSR_LAYER_CH2_WAVES": "0"})):
        path = str(tmp_path / f"{tag}.npz")
        res = subprocess.run([sys.executable, "-c", prog, path], cwd=ROOT, env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=900)
        assert res.returncode == 0, (tag, res.stderr[-2000:])
        outs.append((tag, np.load(path)))
    ref = outs[0][1]
    assert ref["C4_ok"].sum() >= 100 and ref["C2_ok"].sum() >= 100
    for tag, o in outs[1:]:
        for k in ref.files:
            assert np.array_equal(ref[k], o[k]), (tag, k)


def test_reconcile_layered_c4b_full_size_properties(cv, ctx):
    """C4b at full size (N_R = 5e6, 25 frames: one 32-frame tile at one frame per lane, the
    paper's experimental optimum P:408) in the bench's launch configuration: properties that hold
    at any size -- every reconciled frame reproduces Bob's syndromes of every coded slice, no frame
    is an undetected error, flags and counts agree with cvsr_stats, iterations stay in range."""
    cfg = configs.C4b
    codes_l = cfg.build_codes()
    F, n = cfg.frames, cfg.n
    from cvsr_inputs.awgn import torch_quadratures
    from paper_2108_08418_b200.pipeline import SRPipeline
    xd, yd = torch_quadratures(F, n, cfg.gamma, torch.device("cuda:0"))
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, n, F, torch.device("cuda:0"),
                      max_iter=cfg.max_iter, schedule="layered")
    st = pipe.step(xd, yd, want_stats=True)
    torch.cuda.synchronize()
    ok = pipe.frame_ok.cpu().numpy().astype(bool)
    it = pipe.iters.cpu().numpy()
    assert st["frames"] == F and st["frames_ok"] == int(ok.sum()) and ok.all()
    assert st["schedule"] == [0 if c is None else LAYERED for c in codes_l]
    for j, c in enumerate(codes_l):
        if c is None:
            assert (it[:, j] == 0).all()
            continue
        assert ((it[:, j] >= 0) & (it[:, j] <= cfg.max_iter)).all()
        s_a = torch.empty_like(pipe.synd[j])
        cv.cvsr_syndrome(pipe.ctx, pipe.code_h[j], pipe.label_alice, F, j, s_a)
        torch.cuda.synchronize()
        assert (s_a == pipe.synd[j]).all(dim=1).cpu().numpy()[ok].all()
    assert pipe.count_errors()[1] == 0
    pipe.close()
