"""Seeded LDPC code construction (input generator shared by the CUDA path and the oracle).

The paper fixes neither its degree distributions (PAPER.md:392 defers to external
references) nor its construction.  The ensembles here are the
PROPOSED substitutes of SURVEY.md §8(d):

* ``regular(dv, dc)`` -- e.g. the (3,6) code of config C1;
* ``irregular_rate(R)`` -- the edge-perspective variable distribution
  lambda(x) = 0.30013x + 0.28395x^2 + 0.41592x^7 (SURVEY.md §8(d) "Irregular
  ensembles") with check degrees concentrated on two consecutive values so that
  the realised rate is 1 - M/n;
* ``met_low_rate(alpha, beta, dv_core, dc_core)`` -- the MET-style low-rate
  structure of SURVEY.md §8(d) (degree-1 variables + degree-2 type-A checks
  + a core LDPC), used for rates < 0.1.

All constructions are deterministic functions of (ensemble, n, seed).  The
returned :class:`Code` is plain data (CSR by check); it carries no decoder
arithmetic.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Dict, Tuple

import numpy as np

from . import _native

# rate-1/2-optimised BI-AWGN variable-edge distribution
LAMBDA_IRREGULAR: Dict[int, float] = {2: 0.30013, 3: 0.28395, 8: 0.41592}


@dataclasses.dataclass(frozen=True)
class Code:
    """Parity-check matrix H (M x n) in CSR-by-check form."""

    n: int
    m_checks: int
    row_ptr: np.ndarray  # int32[M+1]
    col_idx: np.ndarray  # int32[E], ascending within each row
    name: str = ""

    @property
    def n_edges(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def rate(self) -> float:
        """Realised rate R_j = 1 - M/n (SPEC.md:199 reading, full-rank assumption)."""
        return 1.0 - self.m_checks / self.n

    def digest(self) -> str:
        h = hashlib.sha256()
        h.update(np.int64([self.n, self.m_checks]).tobytes())
        h.update(self.row_ptr.tobytes())
        h.update(self.col_idx.tobytes())
        return h.hexdigest()[:16]

    def dense(self) -> np.ndarray:
        """Dense 0/1 matrix (tiny codes only; test helper)."""
        H = np.zeros((self.m_checks, self.n), dtype=np.uint8)
        for c in range(self.m_checks):
            H[c, self.col_idx[self.row_ptr[c]:self.row_ptr[c + 1]]] = 1
        return H


def from_dense(H: np.ndarray, name: str = "dense") -> Code:
    H = np.asarray(H, dtype=np.uint8)
    M, n = H.shape
    rows = [np.nonzero(H[c])[0].astype(np.int32) for c in range(M)]
    row_ptr = np.zeros(M + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    col_idx = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    return Code(n, M, row_ptr, col_idx, name)


def _i32p(a: np.ndarray):
    import ctypes
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def from_degrees(var_deg: np.ndarray, chk_deg: np.ndarray, seed: int, name: str = "") -> Code:
    var_deg = np.ascontiguousarray(var_deg, dtype=np.int32)
    chk_deg = np.ascontiguousarray(chk_deg, dtype=np.int32)
    n, M = len(var_deg), len(chk_deg)
    E = int(var_deg.sum())
    if E != int(chk_deg.sum()):
        raise ValueError("variable and check degree sums differ")
    row_ptr = np.zeros(M + 1, dtype=np.int32)
    col_idx = np.zeros(E, dtype=np.int32)
    rc = _native.lib().ldpc_configuration_model(n, M, _i32p(var_deg), _i32p(chk_deg),
                                                 seed & 0xFFFFFFFFFFFFFFFF, _i32p(row_ptr), _i32p(col_idx))
    if rc != 0:
        raise RuntimeError(f"ldpc_configuration_model failed ({rc})")
    return Code(n, M, row_ptr, col_idx, name)


def peg_from_degrees(var_deg: np.ndarray, chk_deg: np.ndarray, seed: int, depth: int = 4, name: str = "") -> Code:
    """Progressive-edge-growth construction (host C, `ldpc_peg`): no cycle shorter than
    2 (depth + 2) is closed where the degree targets allow it."""
    var_deg = np.ascontiguousarray(var_deg, dtype=np.int32)
    chk_deg = np.ascontiguousarray(chk_deg, dtype=np.int32)
    n, M = len(var_deg), len(chk_deg)
    E = int(var_deg.sum())
    if E != int(chk_deg.sum()):
        raise ValueError("variable and check degree sums differ")
    row_ptr = np.zeros(M + 1, dtype=np.int32)
    col_idx = np.zeros(E, dtype=np.int32)
    rc = _native.lib().ldpc_peg(n, M, _i32p(var_deg), _i32p(chk_deg), seed & 0xFFFFFFFFFFFFFFFF, depth,
                                _i32p(row_ptr), _i32p(col_idx))
    if rc != 0:
        raise RuntimeError(f"ldpc_peg failed ({rc})")
    return Code(n, M, row_ptr, col_idx, name)


def permutation(n: int, seed: int) -> np.ndarray:
    p = np.zeros(n, dtype=np.int32)
    if _native.lib().ldpc_permutation(n, seed & 0xFFFFFFFFFFFFFFFF, _i32p(p)) != 0:
        raise RuntimeError("ldpc_permutation failed")
    return p


def _node_counts(lam: Dict[int, float], n: int) -> Dict[int, int]:
    """Edge-perspective lambda -> integer node counts summing to n (largest remainder)."""
    inv = {a: l / a for a, l in lam.items()}
    s = sum(inv.values())
    frac = {a: n * v / s for a, v in inv.items()}
    cnt = {a: int(np.floor(f)) for a, f in frac.items()}
    rem = n - sum(cnt.values())
    for a in sorted(frac, key=lambda a: frac[a] - cnt[a], reverse=True)[:rem]:
        cnt[a] += 1
    return cnt


def _two_degree_checks(E: int, M: int) -> np.ndarray:
    d = E // M
    hi = E - d * M  # checks of degree d+1
    deg = np.full(M, d, dtype=np.int32)
    deg[:hi] = d + 1
    return deg


def regular(n: int, dv: int, dc: int, seed: int = 1) -> Code:
    if (n * dv) % dc:
        raise ValueError("n*dv must be divisible by dc")
    M = n * dv // dc
    return from_degrees(np.full(n, dv, np.int32), np.full(M, dc, np.int32), seed,
                        name=f"regular({dv},{dc}) n={n}")


def irregular_rate(n: int, rate: float, seed: int = 1,
                   lam: Dict[int, float] = LAMBDA_IRREGULAR, chain_degree2: bool = True,
                   construction: str = "config", peg_depth: int = 4) -> Code:
    """Irregular code of realised rate 1 - M/n, M = round((1-rate) n).

    chain_degree2 (default): the degree-2 variables form a single path through
    the checks ("staircase"), so the degree-2 subgraph has no cycle.  In a plain
    configuration model with lambda_2 = 0.30 that subgraph has many short
    cycles, i.e. codewords of weight 3..6 supported on degree-2 variables,
    which BP converges to as undetected errors (measured: 4/16 frames of C2's
    S2 slice).  Requires #degree-2 variables < M; at high rates the excess
    degree-2 variables become degree-3.  The remaining sockets are matched by
    the seeded configuration model with duplicate repair.
    """
    cnt = _node_counts(lam, n)
    M = int(round((1.0 - rate) * n))
    if chain_degree2 and cnt.get(2, 0) >= M and 3 in cnt:
        # high rates (M < #degree-2 variables): a cycle-free degree-2 subgraph needs fewer
        # degree-2 variables; move the excess to degree 3 (PROPOSED, R-3)
        excess = cnt[2] - (M - max(1, M // 200))
        cnt[2] -= excess
        cnt[3] += excess
    var_deg = np.concatenate([np.full(c, a, np.int32) for a, c in sorted(cnt.items())])
    var_deg = var_deg[permutation(n, seed ^ 0x5EED)]
    chk_deg = _two_degree_checks(int(var_deg.sum()), M)
    chk_deg = chk_deg[permutation(M, seed ^ 0xC4EC)]
    name = f"irregular R={1 - M / n:.4f} n={n}"
    if construction == "peg":
        return peg_from_degrees(var_deg, chk_deg, seed, peg_depth, name=name + " (PEG)")
    d2 = np.nonzero(var_deg == 2)[0].astype(np.int32)
    if not chain_degree2 or len(d2) == 0 or len(d2) >= M:
        return from_degrees(var_deg, chk_deg, seed, name=name)
    # staircase over a seeded check order: degree-2 var d2[k] joins checks pi[k], pi[k+1]
    pi = permutation(M, seed ^ 0x57A1).astype(np.int32)
    chain_r = np.concatenate([pi[:-1][:len(d2)], pi[1:][:len(d2)]])
    chain_v = np.concatenate([d2, d2])
    chain_cnt = np.bincount(chain_r, minlength=M).astype(np.int32)
    rest_c = chk_deg - chain_cnt
    if np.any(rest_c < 0):
        raise ValueError("check degrees too small for the degree-2 chain")
    rest_v = np.where(var_deg == 2, 0, var_deg).astype(np.int32)
    rest = from_degrees(rest_v, rest_c, seed, name="rest")
    rows_rest = np.repeat(np.arange(M, dtype=np.int32), np.diff(rest.row_ptr))
    r_all = np.concatenate([rows_rest, chain_r])
    v_all = np.concatenate([rest.col_idx, chain_v])
    order = np.lexsort((v_all, r_all))
    row_ptr = np.zeros(M + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum(np.bincount(r_all, minlength=M))
    return Code(n, M, row_ptr, v_all[order].astype(np.int32), name + " (degree-2 chain)")


def met_low_rate(n: int, alpha: float, beta: float, dv_core: int = 3, dc_core: int = 6,
                 seed: int = 1) -> Code:
    """MET-style low-rate code (PROPOSED): rate alpha - beta.

    Variables: n_c = alpha*n core nodes + (n - n_c) degree-1 nodes.  Checks:
    (n - n_c) type-A degree-2 checks {degree-1 var, core var}; each core var
    is in ~ (1-alpha)/alpha type-A checks; plus M_B = beta*n type-B checks
    forming a core LDPC over the core variables with core degrees (dv_core,
    dc_core-ish).  Variable index order: core first, then degree-1.
    """
    n_c = int(round(alpha * n))
    n_1 = n - n_c
    M_B = int(round(beta * n))
    rng_perm = permutation(n_1, seed ^ 0xA11A)
    # type-A: degree-1 var (n_c + i) with core var (perm[i] mod n_c)
    core_of = (rng_perm % n_c).astype(np.int32)
    # core LDPC via configuration model over core vars
    core_vdeg = np.full(n_c, dv_core, np.int32)
    core_cdeg = _two_degree_checks(int(core_vdeg.sum()), M_B)
    core = from_degrees(core_vdeg, core_cdeg, seed, name="core")
    # assemble rows: type-B rows first, then type-A rows (sorted columns)
    rows_B = [core.col_idx[core.row_ptr[c]:core.row_ptr[c + 1]] for c in range(M_B)]
    lens = np.concatenate([np.diff(core.row_ptr), np.full(n_1, 2, np.int32)])
    row_ptr = np.zeros(M_B + n_1 + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum(lens)
    col_idx = np.empty(int(row_ptr[-1]), dtype=np.int32)
    col_idx[:core.n_edges] = core.col_idx
    a = core_of
    b = np.arange(n_c, n, dtype=np.int32)
    pairs = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1).reshape(-1)
    col_idx[core.n_edges:] = pairs
    del rows_B
    return Code(n, M_B + n_1, row_ptr, col_idx,
                name=f"MET alpha={alpha} beta={beta} core({dv_core},{dc_core}) n={n}")


def met_irregular_core(n: int, alpha: float, core_rate: float, seed: int = 1,
                       lam: Dict[int, float] = LAMBDA_IRREGULAR) -> Code:
    """MET-style low-rate code with an IRREGULAR core (PROPOSED, R-2'): rate
    alpha * core_rate.  Variables: n_c = alpha*n core nodes (indices 0..n_c-1) + n - n_c
    degree-1 nodes; checks: the core code irregular_rate(n_c, core_rate, lam) over the core
    nodes, then n - n_c type-A degree-2 checks {degree-1 node, core node}, the core nodes taking
    the degree-1 nodes round-robin (~(1-alpha)/alpha each).  The type-A checks repeat every core
    bit over several channel uses; the core code then works at a rate suited to its ensemble."""
    n_c = int(round(alpha * n))
    n_1 = n - n_c
    core = irregular_rate(n_c, core_rate, seed=seed, lam=lam)
    M_B = core.m_checks
    core_of = (permutation(n_1, seed ^ 0xA11A) % n_c).astype(np.int32)
    lens = np.concatenate([np.diff(core.row_ptr), np.full(n_1, 2, np.int32)])
    row_ptr = np.zeros(M_B + n_1 + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum(lens)
    col_idx = np.empty(int(row_ptr[-1]), dtype=np.int32)
    col_idx[:core.n_edges] = core.col_idx
    b = np.arange(n_c, n, dtype=np.int32)
    col_idx[core.n_edges:] = np.stack([np.minimum(core_of, b), np.maximum(core_of, b)], axis=1).reshape(-1)
    return Code(n, M_B + n_1, row_ptr, col_idx,
                name=f"MET alpha={alpha} irregular core R={core_rate} n={n}")


def csc(code: Code) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(col_ptr[n+1], row_of_edge[E] in CSC order, csr_pos[E] in CSC order)."""
    E = code.n_edges
    rows = np.repeat(np.arange(code.m_checks, dtype=np.int32), np.diff(code.row_ptr))
    order = np.lexsort((rows, code.col_idx))  # by column then row
    col_ptr = np.zeros(code.n + 1, dtype=np.int32)
    np.add.at(col_ptr, code.col_idx + 1, 1)
    col_ptr = np.cumsum(col_ptr).astype(np.int32)
    return col_ptr, rows[order].astype(np.int32), order.astype(np.int32)[:E]


def degree_histograms(code: Code) -> Tuple[Dict[int, int], Dict[int, int]]:
    vdeg = np.bincount(code.col_idx, minlength=code.n)
    cdeg = np.diff(code.row_ptr)
    hv = dict(zip(*np.unique(vdeg, return_counts=True)))
    hc = dict(zip(*np.unique(cdeg, return_counts=True)))
    return {int(k): int(v) for k, v in hv.items()}, {int(k): int(v) for k, v in hc.items()}
