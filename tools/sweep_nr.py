#!/usr/bin/env python3
"""C5: sub-block-size sweep at a fixed number of symbols per GPU.

For N_R = 2^12 .. 2^20 (PAPER.md:102 N_d = floor(N / N_R) sub-blocks), decode
N = 1.25e8 symbols per GPU (1e9 over 8 GPUs) with C4's slice structure and
report throughput, FER, iterations and beta per N_R -- the trade-off of
PAPER.md Section IV measured on B200 instead of modelled with c_h.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from cvsr_inputs import configs  # noqa: E402
from cvsr_inputs.awgn import torch_quadratures  # noqa: E402
from paper_2108_08418_b200 import keyrate as analysis  # noqa: E402  (host-side beta formula)
from paper_2108_08418_b200.pipeline import SRPipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--symbols", type=int, default=configs.C5_SYMBOLS_PER_GPU)
    ap.add_argument("--nr", default=",".join(str(x) for x in configs.C5_NR))
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--schedule", default="layered", choices=["layered", "flooding"])
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for n_r in [int(v) for v in args.nr.split(",")]:
        cfg = configs.c5(n_r)
        frames = max(1, args.symbols // n_r)
        codes_l = cfg.build_codes()
        pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, n_r, frames, dev, cfg.max_iter,
                          schedule=args.schedule)
        x, y = torch_quadratures(frames, n_r, cfg.gamma, dev)
        st = pipe.step(x, y, want_stats=True)
        und = pipe.count_errors()[1]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            pipe.step(x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        rates = [c.rate if c is not None else 0.0 for c in codes_l]
        pi_my, _ = analysis.entropies(cfg.gamma, cfg.m, cfg.delta)
        ok = st["frames_ok"] - und
        print(json.dumps({"n_r": n_r, "frames": frames, "ms_per_step": ms, "schedule": args.schedule,
                          "reconciled_bits_per_s": ok * cfg.m * n_r / (ms * 1e-3),
                          "fer": 1 - st["frames_ok"] / frames, "undetected": und,
                          "mean_iters": [s / max(a, 1) for s, a in zip(st["iters_sum"], st["attempted"])],
                          "beta": analysis.beta(pi_my, cfg.m, rates, cfg.gamma),
                          "goodput_beta_x_1mFER": analysis.beta(pi_my, cfg.m, rates, cfg.gamma) * ok / frames}),
              flush=True)
        pipe.close()
        del x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
