#!/usr/bin/env python3
"""Rate back-off calibration on the GPU.

For each coded slice of a config, try rates R_j = 0.9*cap_j - k*Delta R
(Delta R = 0.05) and measure the per-slice frame-error rate on
`--frames` synthetic frames with the CUDA path; a rate passes when its FER is
at or below --target (a testable surrogate for eps_EC).  Prints
one JSON line per trial.
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


def trial(cfg, frames, seed_frame):
    codes_l = cfg.build_codes()
    dev = torch.device("cuda:0")
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, frames, dev, cfg.max_iter)
    x, y = torch_quadratures(frames, cfg.n, cfg.gamma, dev, first_frame=seed_frame)
    st = pipe.step(x, y, want_stats=True)
    err = pipe.count_errors()
    pipe.close()
    out = {"rates": [round(c.rate, 4) if c is not None else None for c in codes_l], "frames": frames,
           "frames_ok": st["frames_ok"], "undetected": err[1], "slices": {}}
    for j, c in enumerate(codes_l):
        if c is None:
            continue
        a, cv = st["attempted"][j], st["converged"][j]
        out["slices"][j] = {"rate": round(c.rate, 4), "attempted": a, "fer": (1 - cv / a) if a else None,
                            "mean_iters": st["iters_sum"][j] / max(a, 1)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=0, help="0 = the config's frames per GPU")
    ap.add_argument("--grid", default="2:0.406,0.356;3:0.307,0.257,0.207")
    args = ap.parse_args()
    base = configs.CONFIGS[args.config]
    grid = {}
    for part in args.grid.split(";"):
        j, rs = part.split(":")
        grid[int(j)] = [r if r.startswith("met") else float(r) for r in rs.split(",")]
    frames = args.frames or base.frames
    for j, rates in grid.items():
        for r in rates:
            kind = "irregular"
            if isinstance(r, str) and r.startswith("met"):
                kind, r = "met", float(r[3:])
            met = (2 * r, r, 3, 6) if kind == "met" else None
            sl = tuple(dataclasses.replace(s, rate=r, kind=kind, met=met) if s.j == j else s for s in base.slices)
            cfg = dataclasses.replace(base, slices=sl)
            res = trial(cfg, frames, 10_000_000)
            res["vary_slice"] = j
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
