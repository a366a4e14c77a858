#!/usr/bin/env python3
"""Schedule study (CPU, numpy): flooding vs row-layered sum-product on C2's coded-slice codes.

The paper does not fix the BP schedule (SURVEY §8(c) A-8 reads it as
flooding, which is what the CUDA path and the oracle implement).  This tool measures,
on the C2 codes, how many iterations a row-layered schedule (checks greedily coloured
into layers that share no variable; posteriors updated after every layer) needs
against flooding on the same frames, to size a possible next-round decoder.

Channel: a BI-AWGN surrogate of each slice (u ~ Bernoulli(1/2), syndrome s = H u,
LLR = 2y/sigma^2), sigma chosen so that R / C_BIAWGN(sigma) equals the slice's
efficiency R_j / cap_j on C2 (0.356/0.452 and 0.257/0.341).  This is a
stand-alone numpy decoder (not the oracle, not the CUDA path).

  python tools/layered_study.py [frames]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from cvsr_inputs import configs  # noqa: E402

Q_MAX = 40.0


def phi(x):
    x = np.clip(x, 1e-12, Q_MAX)
    return -np.log(np.tanh(0.5 * x))


def biawgn_capacity(sigma, n=200001):
    t = np.linspace(-12, 12, n)
    y = 1.0 + sigma * t
    w = np.exp(-0.5 * t * t) / np.sqrt(2 * np.pi)
    return 1.0 - float(np.sum(w * np.logaddexp(0.0, -2.0 * y / sigma ** 2)) * (t[1] - t[0]) / np.log(2))


def sigma_for(capacity):
    lo, hi = 0.1, 5.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if biawgn_capacity(mid) > capacity:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def layers(code):
    """Greedy colouring: checks of one layer share no variable."""
    used = np.zeros(code.n, np.int64)
    colour = np.empty(code.m_checks, np.int64)
    rp, ci = code.row_ptr, code.col_idx
    for c in range(code.m_checks):
        vs = ci[rp[c]:rp[c + 1]]
        mask = int(np.bitwise_or.reduce(used[vs])) if len(vs) else 0
        k = 0
        while mask >> k & 1:
            k += 1
        colour[c] = k
        used[vs] |= 1 << k
    return colour


def cn_update(q, chk_of_edge, seg_starts, s_c):
    """Sum-product check update for the edges (F, E') grouped by check (reduceat segments)."""
    a = np.abs(q)
    p = phi(a)
    tot = np.add.reduceat(p, seg_starts, axis=1)
    neg = np.add.reduceat((q < 0).astype(np.int64), seg_starts, axis=1) + s_c
    mag = phi(tot[:, chk_of_edge] - p)
    sgn = 1 - 2 * ((neg[:, chk_of_edge] - (q < 0)) & 1)
    return sgn * mag


def syndrome_ok(code, hard, s):
    rp = code.row_ptr
    par = np.add.reduceat(hard[:, code.col_idx].astype(np.int64), rp[:-1], axis=1) & 1
    return np.all(par == s, axis=1)


def decode(code, llr, s, schedule, colour=None, max_iter=100):
    F = llr.shape[0]
    E = code.n_edges
    rp, ci = code.row_ptr, code.col_idx
    chk = np.repeat(np.arange(code.m_checks), np.diff(rp))
    r = np.zeros((F, E))
    post = llr.copy()
    iters = np.full(F, -1)
    active = np.ones(F, bool)
    if schedule == "layered":
        groups = []
        for L in range(int(colour.max()) + 1):
            cs = np.nonzero(colour == L)[0]
            eidx = np.concatenate([np.arange(rp[c], rp[c + 1]) for c in cs])
            seg = np.concatenate([[0], np.cumsum(np.diff(rp)[cs])[:-1]])
            groups.append((cs, eidx, np.repeat(np.arange(len(cs)), np.diff(rp)[cs]), seg))
    for k in range(max_iter + 1):
        ok = syndrome_ok(code, post < 0, s) & active
        iters[ok] = k
        active &= ~ok
        if k == max_iter or not active.any():
            break
        a = np.nonzero(active)[0]
        if schedule == "flooding":
            q = np.clip(post[a][:, ci] - r[a], -Q_MAX, Q_MAX)
            rn = cn_update(q, chk, rp[:-1], s[a])
            r[a] = rn
            post[a] = llr[a] + np.stack([np.bincount(ci, rn[i], code.n) for i in range(len(a))])
        else:
            for cs, eidx, loc, seg in groups:
                vs = ci[eidx]
                pa = post[a]
                q = np.clip(pa[:, vs] - r[a][:, eidx], -Q_MAX, Q_MAX)
                rn = cn_update(q, loc, seg, s[a][:, cs])
                pa[:, vs] = q + rn
                post[a] = pa
                ra = r[a]
                ra[:, eidx] = rn
                r[a] = ra
    return iters


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    cfg = configs.C2
    codes_l = cfg.build_codes()
    eff = {2: 0.356 / 0.4520, 3: 0.257 / 0.3414}
    rng = np.random.default_rng(7)
    for j, code in enumerate(codes_l):
        if code is None:
            continue
        sigma = sigma_for(code.rate / eff[j])
        u = rng.integers(0, 2, (F, code.n)).astype(np.uint8)
        y = (1.0 - 2.0 * u) + sigma * rng.standard_normal((F, code.n))
        llr = np.clip(2.0 * y / sigma ** 2, -Q_MAX, Q_MAX)
        s = np.add.reduceat(u[:, code.col_idx].astype(np.int64), code.row_ptr[:-1], axis=1) & 1
        t0 = time.time()
        colour = layers(code)
        t1 = time.time()
        it_f = decode(code, llr, s, "flooding")
        it_l = decode(code, llr, s, "layered", colour)
        print(json.dumps({"slice": j, "rate": round(code.rate, 4), "E_over_n": code.n_edges / code.n,
                          "sigma": round(sigma, 4), "frames": F, "layers": int(colour.max()) + 1,
                          "colour_s": round(t1 - t0, 2),
                          "flooding_iters": it_f.tolist(), "layered_iters": it_l.tolist(),
                          "mean_flooding": float(np.mean(it_f[it_f >= 0])) if (it_f >= 0).any() else None,
                          "mean_layered": float(np.mean(it_l[it_l >= 0])) if (it_l >= 0).any() else None}),
              flush=True)


if __name__ == "__main__":
    main()
