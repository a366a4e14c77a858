#!/usr/bin/env python3
"""C4's S2 slice (capacity 0.167): FER / iterations / step time of candidate low-rate ensembles
on the GPU at the back-off ladder's rates (0.166, 0.116), S3 = 0.598 and S4 = 0.441 fixed.

    python tools/try_s2.py --frames 1000
"""
import argparse
import dataclasses
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from cvsr_inputs import configs  # noqa: E402

spec = importlib.util.spec_from_file_location("backoff", os.path.join(ROOT, "tools", "backoff.py"))
bo = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bo)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=1000)
    ap.add_argument("--rates", default="0.116,0.166")
    ap.add_argument("--core-rates", default="0.4,0.5,0.6")
    ap.add_argument("--no-met", action="store_true")
    args = ap.parse_args()
    base = configs.C4
    cands = []
    for r in (float(v) for v in args.rates.split(",")):
        for rc in (float(v) for v in args.core_rates.split(",")):
            cands.append(("met_irr", r, (round(r / rc, 6), rc, 0, 0)))
        if not args.no_met:
            cands.append(("met", r, (round(2 * r, 6), r, 3, 6)))
    for kind, r, met in cands:
        sl = tuple(configs.SliceSpec(2, kind, r, met) if s.j == 2 else s for s in base.slices)
        cfg = dataclasses.replace(base, slices=sl)
        codes_l = cfg.build_codes()
        res = bo.test(cfg, codes_l, 2, args.frames, base.frames)
        print(json.dumps({"kind": kind, "rate": r, "met": met, "realised": codes_l[2].rate,
                          "max_dc": int(max(codes_l[2].row_ptr[1:] - codes_l[2].row_ptr[:-1])),
                          "edges": codes_l[2].n_edges, **res}), flush=True)


if __name__ == "__main__":
    main()
