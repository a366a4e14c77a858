#!/usr/bin/env python3
"""Variable-degree distribution design by Gaussian-approximation density evolution (NEXT-1/NEXT-2).

For a slice of rate R decoded at slice capacity C (the BI-AWGN channel of equal
capacity stands in for the slice channel), search lambda(x) on a fixed degree
set to minimise the modelled decoder traffic per symbol

    cost = D_GA(sigma_C, eps = 1/n) * (16 E/n + 4)      [bytes per symbol]

(D_GA: GA iterations until the decision error is below 1/n, PAPER.md eq:rob2
with reading A-19; 16 B per edge and 4 B per variable per flooding iteration
is this implementation's traffic).  rho is concentrated on two
consecutive degrees that realise R.  Constraint: the degree-2 variables must
fit the cycle-free staircase (fewer than M = (1 - R) n).

  python tools/design_ensemble.py --rate 0.257 --cap 0.3414 --n 65536
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
from scipy import optimize  # noqa: E402

from paper_2108_08418_b200 import keyrate as K  # noqa: E402

DEGREES = (2, 3, 4, 5, 6, 8, 10, 12)


def rho_for(lam: dict, rate: float):
    """Two consecutive check degrees (edge perspective) realising `rate` for lambda."""
    s_lam = sum(l / a for a, l in lam.items())          # = n / E
    s_rho = (1.0 - rate) * s_lam                         # = M / E = sum rho_b / b
    davg = 1.0 / s_rho                                    # mean check degree (node perspective)
    b = int(math.floor(davg))
    if b < 2:
        return None
    # node fractions f_b, f_(b+1) with mean davg; edge perspective rho_b = b f_b / davg
    f_hi = davg - b
    rho = {b: b * (1 - f_hi) / davg}
    if f_hi > 1e-9:
        rho[b + 1] = (b + 1) * f_hi / davg
    return rho


_SIGMA = {}


def evaluate(lam: dict, rate: float, cap: float, n: int, max_iter: int = 200):
    rho = rho_for(lam, rate)
    if rho is None:
        return None
    e_per_n = 1.0 / sum(l / a for a, l in lam.items())
    frac2 = (lam.get(2, 0.0) / 2.0) * e_per_n            # degree-2 variables per symbol
    if frac2 >= (1.0 - rate):
        return None
    if cap not in _SIGMA:
        _SIGMA[cap] = K.biawgn_sigma_for_capacity(cap)
    sigma = _SIGMA[cap]
    d = K.ga_iterations(2.0 / sigma ** 2, lam, rho, 1.0 / n, max_iter)
    if d > max_iter:
        return None
    return {"lam": lam, "rho": rho, "E_per_n": e_per_n, "D_GA": d, "cost": d * (16 * e_per_n + 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, required=True)
    ap.add_argument("--cap", type=float, required=True)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--degrees", default=",".join(map(str, DEGREES)))
    args = ap.parse_args()
    degrees = tuple(int(d) for d in args.degrees.split(","))
    ref = evaluate({2: 0.30013, 3: 0.28395, 8: 0.41592}, args.rate, args.cap, args.n)
    print(json.dumps({"reference": ref}), flush=True)

    def lam_of(w):
        w = np.maximum(w, 0.0)
        if w.sum() <= 0:
            return None
        w = w / w.sum()
        return {a: float(x) for a, x in zip(degrees, w) if x > 1e-4}

    def f(w):
        lam = lam_of(w)
        if lam is None:
            return 1e9
        r = evaluate(lam, args.rate, args.cap, args.n)
        return 1e9 if r is None else r["cost"]

    res = optimize.differential_evolution(f, [(0.0, 1.0)] * len(degrees), seed=args.seed, maxiter=args.iters,
                                          popsize=12, tol=1e-4, polish=False)
    best = evaluate(lam_of(res.x), args.rate, args.cap, args.n)
    print(json.dumps({"best": best}), flush=True)


if __name__ == "__main__":
    main()
