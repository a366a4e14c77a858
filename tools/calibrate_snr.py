#!/usr/bin/env python3
"""Lowest SNR at which a fixed-rate config decodes (FER <= target), on the GPU.

Used for C3 (rate ~0.02 MET-style code, "low-SNR LEO channel"): the config fixes
the rate, so the operating SNR is the free parameter (the converse of the rate
back-off of PAPER.md:394).  Prints one JSON line per gamma.
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from cvsr_inputs import configs  # noqa: E402
from cvsr_inputs.awgn import torch_quadratures  # noqa: E402
from paper_2108_08418_b200.pipeline import SRPipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--gammas", default="0.08,0.10,0.12,0.15,0.20")
    ap.add_argument("--frames", type=int, default=0)
    args = ap.parse_args()
    base = configs.CONFIGS[args.config]
    codes_l = base.build_codes()
    dev = torch.device("cuda:0")
    for g in [float(v) for v in args.gammas.split(",")]:
        cfg = dataclasses.replace(base, gamma=g)
        F = args.frames or cfg.frames
        pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, F, dev, cfg.max_iter)
        x, y = torch_quadratures(F, cfg.n, g, dev, first_frame=20_000_000)
        st = pipe.step(x, y, want_stats=True)
        und = pipe.count_errors()[1]
        pipe.close()
        j = [i for i, c in enumerate(codes_l) if c is not None]
        print(json.dumps({"gamma": g, "frames": F, "fer": 1 - st["frames_ok"] / F, "undetected": und,
                          "mean_iters": [st["iters_sum"][i] / max(st["attempted"][i], 1) for i in j]}), flush=True)


if __name__ == "__main__":
    main()
