#!/usr/bin/env python3
"""Rate back-off against the code database, on the GPU (reading R-2' of DESIGN.md).

For each slice S_j in decode order (PAPER.md:394 steps 1-3):
  1) select the code whose rate is closest to (and not above) the slice capacity cap_j
     (reading A-6; R_0 = floor(1000 cap_j) / 1000) -- or 0 (disclosed) below the database floor
     0.01;
  2) test its frame-error rate on synthetic frames with the CUDA path (layered BP, the bench's
     schedule): the test passes when no frame fails in `--frames` (so the 95 % upper bound of the
     FER is <= 3/frames; a testable surrogate for eps_EC) and no frame is an
     undetected error;
  3) if it fails, R_j -= Delta R = 0.05 and go back to 2); otherwise mark the code "good" and
     continue with the next slice (earlier slices use their good codes).
Families (PAPER.md:392 uses MET codes below R = 0.1 and irregular codes above; our PROPOSED
substitutes, reading A-7): for R < 0.1 the MET-style code (degree-1 variables, degree-2
type-A checks, (3,6) core: alpha = 2R, beta = R); for R >= 0.1 the irregular code first and, if
it fails (up to R = 0.25), the MET-style codes of the same rate -- with an irregular core of rate
0.3, 0.35, 0.4 and 0.5 ("met_irr", alpha = R / core rate), then with the (3,6) core -- before
backing off.  When several families pass at a rate the one with the least decoding work (edges x
mean iterations) is marked good.

    python tools/backoff.py --config C4 --frames 2000 [--write]

prints one JSON line per trial and (--write) stores every trial in cvsr_inputs/codebook.json.
"""
import argparse
import dataclasses
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from cvsr_inputs import codebook, configs  # noqa: E402
from paper_2108_08418_b200 import keyrate  # noqa: E402  (host fp64 formulas)

DELTA_R = 0.05
FLOOR = 0.01


MET_IRR_CORE_RATES = (0.3, 0.35, 0.4, 0.5)


def families(r):
    """Families tried at rate r, in order (PAPER.md:392 reading)."""
    if r < 0.1:
        return ["met"]
    if r <= 0.25:
        return ["irregular"] + [f"met_irr{rc}" for rc in MET_IRR_CORE_RATES] + ["met"]
    return ["irregular"]


def entry_for(cfg, j, family, rate, seed):
    if family == "met":
        params = {"rate": rate, "alpha": round(2 * rate, 6), "beta": round(rate, 6), "dv_core": 3, "dc_core": 6}
    elif family.startswith("met_irr"):
        rc = float(family[len("met_irr"):])
        params = {"rate": rate, "alpha": round(rate / rc, 6), "core_rate": rc}
        family = "met_irr"
    else:
        params = {"rate": rate}
    return {"config": cfg.name, "slice": j, "n": cfg.n, "family": family, "params": params, "seed": seed}


def test(cfg, codes_l, j, frames, batch):
    """FER of slice j over `frames` frames (batches of the config's frames per GPU)."""
    import torch
    from cvsr_inputs.awgn import torch_quadratures
    from paper_2108_08418_b200.pipeline import SRPipeline
    dev = torch.device("cuda:0")
    pipe = SRPipeline(cfg.m, cfg.edges(), codes_l, cfg.order, cfg.sigma_n, cfg.n, batch, dev, cfg.max_iter,
                      schedule="layered")
    att = conv = it = und = 0
    done = 0
    t0 = time.time()
    while done < frames:
        x, y = torch_quadratures(batch, cfg.n, cfg.gamma, dev, first_frame=20_000_000 + done)
        st = pipe.step(x, y, want_stats=True)
        att += st["attempted"][j]
        conv += st["converged"][j]
        it += st["iters_sum"][j]
        und += pipe.count_errors()[1]
        done += batch
    pipe.close()
    return {"frames": done, "attempted": att, "failed": att - conv, "fer": (att - conv) / max(att, 1),
            "mean_iters": it / max(att, 1), "undetected": und, "seconds": round(time.time() - t0, 1)}


def ladder(order, caps, trial):
    """The back-off of PAPER.md:394 for the slices in decode `order` with capacities `caps`:
    trial(j, family, rate, chosen) -> (passed, work) runs the failure test of slice j's candidate
    code given the good codes `chosen` of the earlier slices (work = edges x mean iterations).  At
    the highest rate where any family passes, the passing family with the least work is chosen.
    Returns (chosen, trials): chosen[j] = (family, rate) or None (disclosed), trials = [(j, family,
    rate, passed)] in order."""
    chosen, trials = {}, []
    for j in order:
        r = math.floor(1000 * caps[j]) / 1000
        while True:
            if r < FLOOR:
                chosen[j] = None
                break
            best = None
            for fam in families(r):
                ok, work = trial(j, fam, r, dict(chosen))
                trials.append((j, fam, r, ok))
                if ok and (best is None or work < best[1]):
                    best = (fam, work)
            if best is not None:
                chosen[j] = (best[0], r)
                break
            r = round(r - DELTA_R, 3)
    return chosen, trials


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--frames", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=configs.CODE_SEED)
    ap.add_argument("--write", action="store_true")
    args = ap.parse_args()
    base = configs.CONFIGS[args.config]
    caps = keyrate.slice_capacities(base.gamma, base.m, base.delta, base.order)
    entries = []

    def trial(j, fam, r, chosen):
        slices = []
        for s in base.slices:
            if s.j == j:
                slices.append(_spec(s.j, fam, r))
            elif s.j in chosen:
                slices.append(_spec(s.j, *chosen[s.j]) if chosen[s.j] else dataclasses.replace(s, kind="disclosed"))
            else:
                slices.append(s)
        cfg = dataclasses.replace(base, slices=tuple(slices))
        codes_l = cfg.build_codes(seed=args.seed)
        res = test(cfg, codes_l, j, args.frames, base.frames)
        ok = res["failed"] == 0 and res["undetected"] == 0
        e = entry_for(cfg, j, fam, r, args.seed + 17 * j)
        e["digest"] = codes_l[j].digest()
        e["realised_rate"] = codes_l[j].rate
        e["test"] = res
        e["status"] = "good" if ok else "failed"
        e["cap"] = float(caps[j])
        e["work"] = codes_l[j].n_edges * res["mean_iters"]
        entries.append(e)
        print(json.dumps(e), flush=True)
        return ok, e["work"]

    chosen, _ = ladder(base.order, caps, trial)
    for e in entries:  # only the chosen code of each slice is "good"; other passing ones "passed"
        c = chosen.get(e["slice"])
        picked = c is not None and e["params"]["rate"] == c[1] and (
            e["family"] == c[0] or (c[0].startswith("met_irr") and e["family"] == "met_irr"
                                    and abs(e["params"].get("core_rate", -1) - float(c[0][7:])) < 1e-9))
        if e["status"] == "good" and not picked:
            e["status"] = "passed"
    for j in base.order:
        if chosen.get(j) is None:
            print(json.dumps({"slice": j, "cap": caps[j], "disclosed": True}), flush=True)
    rates = [0.0 if chosen.get(j) is None else chosen[j][1] for j in range(base.m)]
    pi_my, _ = keyrate.entropies(base.gamma, base.m, base.delta)
    beta = keyrate.beta(pi_my, base.m, rates, base.gamma)
    summary = {"config": base.name, "rates": rates, "beta": beta,
               "families": [None if chosen.get(j) is None else chosen[j][0] for j in range(base.m)]}
    print(json.dumps(summary), flush=True)
    if args.write:
        old = [e for e in codebook.load() if e["config"] != base.name]
        codebook.save(old + entries, meta={"procedure": "tools/backoff.py (PAPER.md:394, DESIGN.md R-2')",
                                           "last_summary": summary})


def _spec(j, family, rate):
    if family == "met":
        return configs.SliceSpec(j, "met", rate, (round(2 * rate, 6), round(rate, 6), 3, 6))
    if family.startswith("met_irr"):
        rc = float(family[len("met_irr"):])
        return configs.SliceSpec(j, "met_irr", rate, (round(rate / rc, 6), rc, 0, 0))
    return configs.SliceSpec(j, "irregular", rate)


if __name__ == "__main__":
    main()
