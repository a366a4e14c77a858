import os, sys, subprocess, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
if len(sys.argv) > 1:
    import torch
    import oracle
    from cvsr_inputs import awgn, codes
    from paper_2108_08418_b200 import cvsr
    code = codes.regular(1024, 3, 6, seed=1)
    sigma = awgn.biawgn_sigma(0.5, 1.5)
    u, y = awgn.biawgn(600, 1024, sigma, seed=21)
    llr = np.clip(2.0 * y.astype(np.float64) / sigma ** 2, -40, 40).astype(np.float32)
    synd = oracle.syndrome(code, u, 0)
    ctx = cvsr.cvsr_ctx_create(0, torch.cuda.current_stream())
    h = cvsr.cvsr_code_load(ctx, code.n, code.m_checks, code.row_ptr, code.col_idx)
    F = 600
    bits = torch.empty((F, 32), dtype=torch.int32, device="cuda")
    conv = torch.empty(F, dtype=torch.uint8, device="cuda")
    it = torch.empty(F, dtype=torch.int32, device="cuda")
    cvsr.cvsr_decode(ctx, h, torch.from_numpy(llr).cuda(), torch.from_numpy(synd.view(np.int32)).cuda(), F,
                     cvsr.decode_opts(100, 40.0), bits, conv, it)
    cvsr.cvsr_ctx_sync(ctx)
    np.savez(sys.argv[1], bits=bits.cpu().numpy(), conv=conv.cpu().numpy(), it=it.cpu().numpy())
else:
    res = {}
    for f in ("0", "1"):
        out = f"/tmp/dc_{f}.npz"
        r = subprocess.run([sys.executable, __file__, out], env=dict(os.environ, CVSR_COMPACT=f), capture_output=True, text=True)
        print(f, r.returncode, r.stderr[-500:])
        res[f] = np.load(out)
    a, b = res["0"], res["1"]
    for key in ("bits", "conv", "it"):
        d = np.nonzero(np.any((a[key] != b[key]).reshape(600, -1), axis=1))[0]
        print(key, "mismatch frames", len(d), d[:20])
    d = np.nonzero(a["it"] != b["it"])[0]
    print("iters a", a["it"][d[:20]], "b", b["it"][d[:20]])
    print("iters hist a", np.bincount(a["it"])[:60])
