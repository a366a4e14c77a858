#!/usr/bin/env python3
"""C1: decoder-only (3,6) n = 1024 at E_b/N_0 = 1.5 dB (excluded from the HBM bar).

The working set (3 MB) is L2-resident, so this case is latency/launch bound: report
the time per decode call, FER, mean iterations, edge-iterations/s and the kernel
launches per call, for the configured 100 frames and for larger batches.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from cvsr_inputs import awgn, codes, configs  # noqa: E402
from paper_2108_08418_b200 import cvsr  # noqa: E402


def main():
    c1 = configs.C1
    code = codes.regular(c1["n"], c1["dv"], c1["dc"], seed=1)
    sigma = awgn.biawgn_sigma(0.5, c1["ebn0_db"])
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream()
    ctx = cvsr.cvsr_ctx_create(0, stream)
    h = cvsr.cvsr_code_load(ctx, code.n, code.m_checks, code.row_ptr, code.col_idx)
    opts = cvsr.decode_opts(c1["max_iter"], 40.0)
    for F in (c1["frames"], 1000, 10000):
        u, y = awgn.biawgn(F, code.n, sigma)
        # Bob's syndromes from the transmitted bits (the library's syndrome kernel on label bytes)
        lab = torch.from_numpy(u.astype(np.uint8)).to(dev)
        synd = torch.empty((F, (code.m_checks + 31) // 32), dtype=torch.int32, device=dev)
        cvsr.cvsr_syndrome(ctx, h, lab, F, 0, synd)
        yd = torch.from_numpy(y).to(dev)
        llr = torch.empty_like(yd)
        bits = torch.empty((F, (code.n + 31) // 32), dtype=torch.int32, device=dev)
        conv = torch.empty(F, dtype=torch.uint8, device=dev)
        iters = torch.empty(F, dtype=torch.int32, device=dev)

        def run():
            cvsr.cvsr_llr_biawgn(ctx, yd, y.size, sigma ** 2, 40.0, llr)
            cvsr.cvsr_decode(ctx, h, llr, synd, F, opts, bits, conv, iters)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        l0 = cvsr.cvsr_ctx_launch_count(ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 20
        e0.record(stream)
        for _ in range(K):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        it = iters.cpu().numpy()
        cv = conv.cpu().numpy().astype(bool)
        edge_it = float(np.sum(np.maximum(it, 0) + 1)) * code.n_edges
        print(json.dumps({"config": "C1", "frames": F, "ms_per_decode": ms, "fer": 1 - cv.mean(),
                          "mean_iters_converged": float(it[cv].mean()) if cv.any() else None,
                          "edge_iterations_per_s": edge_it / (ms * 1e-3),
                          "info_bits_per_s": F * code.n * 0.5 / (ms * 1e-3),
                          "launches_per_decode": (cvsr.cvsr_ctx_launch_count(ctx) - l0) / K}), flush=True)
    cvsr.cvsr_code_free(h)
    cvsr.cvsr_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
