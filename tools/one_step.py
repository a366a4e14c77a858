#!/usr/bin/env python3
"""Run exactly ONE bench step (Bob + Alice of one batch) of a config on cuda:0 and print its
statistics as JSON -- the command to put under `ncu` when every launch of one step is wanted
(e.g. the DRAM bytes of all k_layer launches, tools/ncu_traffic.py).

    python tools/one_step.py [--config C4] [--schedule layered] [--frames F]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--schedule", default="layered")
    ap.add_argument("--frames", type=int, default=0)
    a = ap.parse_args()
    import torch
    from cvsr_inputs import configs
    from cvsr_inputs.awgn import torch_quadratures
    from paper_2108_08418_b200.pipeline import SRPipeline
    cfg = configs.CONFIGS[a.config]
    F = a.frames or cfg.frames
    cl = cfg.build_codes()
    dev = torch.device("cuda:0")
    x, y = torch_quadratures(F, cfg.n, cfg.gamma, dev)
    pipe = SRPipeline(cfg.m, cfg.edges(), cl, cfg.order, cfg.sigma_n, cfg.n, F, dev, cfg.max_iter, cfg.q_max,
                      schedule=a.schedule)
    torch.cuda.synchronize()
    st = pipe.step(x, y, want_stats=True)
    torch.cuda.synchronize()
    E = [c.n_edges if c is not None else 0 for c in cl]
    print(json.dumps({"config": a.config, "schedule": a.schedule, "frames": F, "n": cfg.n,
                      "edge_frames": int(sum(st["edge_iters"])), "iters_sum": st["iters_sum"],
                      "frames_ok": st["frames_ok"], "E": E, "schedule_per_slice": st["schedule"]}))
    pipe.close()


if __name__ == "__main__":
    main()
