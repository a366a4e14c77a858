#!/usr/bin/env python3
"""Decode C2 with alternative variable-degree distributions for the coded slices and report
FER, undetected errors, mean iterations and the step time (tools/design_ensemble.py output).

  python tools/try_ensemble.py C2 '{"2": {"2": 0.23, "3": 0.62, ...}, "3": {...}}'
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from cvsr_inputs import configs  # noqa: E402
from cvsr_inputs.awgn import torch_quadratures  # noqa: E402
from paper_2108_08418_b200.pipeline import SRPipeline  # noqa: E402


def run(cfg, label, steps=5, first_frame=0):
    codes_l = cfg.build_codes()
    dev = torch.device("cuda:0")
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, cfg.frames, dev, cfg.max_iter)
    x, y = torch_quadratures(cfg.frames, cfg.n, cfg.gamma, dev, first_frame=first_frame)
    st = pipe.step(x, y, want_stats=True, key=(99, 98, 97))
    und = pipe.count_errors()[1]
    it = pipe.iters.cpu().numpy()
    for _ in range(2):
        pipe.step(x, y, key=(99, 98, 97))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pipe.step(x, y, key=(99, 98, 97))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ok = int(pipe.verified.sum().item())
    print(json.dumps({"label": label, "frames": cfg.frames, "first_frame": first_frame, "ms_per_step": ms,
                      "verified": ok, "fer": 1 - st["frames_ok"] / cfg.frames, "undetected": und,
                      "bits_per_s": ok * cfg.m * cfg.n / (ms * 1e-3),
                      "mean_iters": [float(np.mean(it[:, j][it[:, j] >= 0])) if (it[:, j] >= 0).any() else None
                                     for j in range(cfg.m)],
                      "max_iters": [int(it[:, j].max()) for j in range(cfg.m)],
                      "E": [c.n_edges if c is not None else 0 for c in codes_l]}), flush=True)
    pipe.close()


def main():
    base = configs.CONFIGS[sys.argv[1]]
    lams = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    run(base, f"{base.name} reference")
    slices = tuple(dataclasses.replace(s, lam=tuple(sorted((int(a), float(w)) for a, w in lams[str(s.j)].items())))
                   if str(s.j) in lams else s for s in base.slices)
    cfg = dataclasses.replace(base, slices=slices)
    for k in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):  # disjoint batches for the FER estimate
        run(cfg, f"{base.name} designed", first_frame=k * base.frames)


if __name__ == "__main__":
    main()
