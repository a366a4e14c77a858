import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2108_08418_b200 import cvsr as cv
from cvsr_inputs import codes, awgn
import oracle
code = codes.regular(1024, 3, 6, seed=1)
F = int(sys.argv[1]) if len(sys.argv) > 1 else 45
sigma = awgn.biawgn_sigma(0.5, 1.5)
u, y = awgn.biawgn(F, code.n, sigma, seed=7)
llr = np.clip(2.0 * y.astype(np.float64) / sigma ** 2, -40, 40).astype(np.float32)
synd = oracle.syndrome(code, u, 0)
ctx = cv.cvsr_ctx_create(0, torch.cuda.current_stream())
h = cv.cvsr_code_load(ctx, code.n, code.m_checks, code.row_ptr, code.col_idx)
r = torch.empty((F, code.n_edges), dtype=torch.float32, device="cuda")
post = torch.empty((F, code.n), dtype=torch.float32, device="cuda")
try:
    cv.cvsr_decode_trace(ctx, h, torch.from_numpy(llr).cuda(), torch.from_numpy(synd.view(np.int32)).cuda(), F, 1, 40.0, r, post, flags=2)
    cv.cvsr_ctx_sync(ctx)
    print("ok", F)
except Exception as e:
    print("ERR", F, e)
