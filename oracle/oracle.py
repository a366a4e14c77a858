"""ctypes marshalling for the fp64 C oracle (cvsr_oracle.c).  TEST INFRASTRUCTURE ONLY.

Argument marshalling only; every computation happens in cvsr_oracle.c, whose
functions cite the PAPER.md passage they follow.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cvsr_oracle.c")
_LIB = os.path.join(_HERE, "libcvsr_oracle.so")
_lock = threading.Lock()
_lib = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (fp64, no fast-math, OpenMP over frames)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp",
                               "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.orc_num_threads.restype = ctypes.c_int
            L.orc_quantise.argtypes = [ctypes.c_int32, _f32p, _f32p, ctypes.c_int64, _u8p]
            L.orc_slice_bits.argtypes = [_u8p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _u32p]
            L.orc_syndrome.argtypes = [ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _u8p,
                                       ctypes.c_int32, ctypes.c_int32, _u32p]
            L.orc_llr_slice.argtypes = [ctypes.c_int32, _f32p, ctypes.c_double, _f32p, ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, _u8p,
                                        ctypes.c_double, _f64p]
            L.orc_llr_biawgn.argtypes = [_f32p, ctypes.c_int64, ctypes.c_double, ctypes.c_double, _f64p]
            L.orc_bp_decode.argtypes = [ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _f64p, _u32p,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _u32p, _u8p, _i32p]
            L.orc_bp_trace.argtypes = [ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _f64p, _u32p,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _f64p, _f64p]
            L.orc_layers.argtypes = [ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _i32p]
            L.orc_bp_layered.argtypes = [ctypes.c_int32, ctypes.c_int32, _i32p, _i32p, _f64p, _u32p,
                                         ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int,
                                         _u32p, _u8p, _i32p, _f64p, _f64p]
            L.orc_reconcile.argtypes = [ctypes.c_int32, ctypes.c_int32, _i32p, ctypes.POINTER(_i32p),
                                        ctypes.POINTER(_i32p), _i32p, _f32p, ctypes.c_double, _f32p,
                                        ctypes.POINTER(_u32p), ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int32, _u8p, _u8p, _i32p]
            for name in ("orc_quantise", "orc_slice_bits", "orc_syndrome", "orc_llr_slice",
                         "orc_llr_biawgn", "orc_bp_decode", "orc_bp_trace", "orc_reconcile", "orc_layers", "orc_bp_layered"):
                getattr(L, name).restype = ctypes.c_int
            _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _chk(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} rejected its arguments ({rc})")


def num_threads() -> int:
    return int(_load().orc_num_threads())


def words(bits: int) -> int:
    return (bits + 31) // 32


def quantise(edges: np.ndarray, y: np.ndarray) -> np.ndarray:
    edges = np.ascontiguousarray(edges, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    m = int(round(np.log2(len(edges) + 1)))
    out = np.empty(y.shape, np.uint8)
    _chk(_load().orc_quantise(m, _p(edges, _f32p), _p(y, _f32p), y.size, _p(out, _u8p)), "quantise")
    return out


def slice_bits(label: np.ndarray, j: int) -> np.ndarray:
    label = np.ascontiguousarray(label, np.uint8)
    F, n = label.shape
    out = np.empty((F, words(n)), np.uint32)
    _chk(_load().orc_slice_bits(_p(label, _u8p), F, n, j, _p(out, _u32p)), "slice_bits")
    return out


def syndrome(code, label: np.ndarray, j: int) -> np.ndarray:
    label = np.ascontiguousarray(label, np.uint8)
    F, n = label.shape
    out = np.empty((F, words(code.m_checks)), np.uint32)
    _chk(_load().orc_syndrome(n, code.m_checks, _p(code.row_ptr, _i32p), _p(code.col_idx, _i32p),
                              _p(label, _u8p), F, j, _p(out, _u32p)), "syndrome")
    return out


def llr_slice(edges: np.ndarray, sigma_n: float, x: np.ndarray, j: int, known_mask: int = 0,
              known_label: Optional[np.ndarray] = None, llr_max: float = 40.0) -> np.ndarray:
    edges = np.ascontiguousarray(edges, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    x2 = x.reshape(-1, x.shape[-1]) if x.ndim > 1 else x.reshape(1, -1)
    F, n = x2.shape
    m = int(round(np.log2(len(edges) + 1)))
    kl = None
    if known_mask:
        kl = np.ascontiguousarray(known_label, np.uint8).reshape(F, n)
    out = np.empty((F, n), np.float64)
    _chk(_load().orc_llr_slice(m, _p(edges, _f32p), float(sigma_n), _p(x2, _f32p), F, n, j,
                               known_mask, _p(kl, _u8p) if kl is not None else None,
                               float(llr_max), _p(out, _f64p)), "llr_slice")
    return out.reshape(x.shape)


def llr_biawgn(y: np.ndarray, sigma2: float, llr_max: float = 40.0) -> np.ndarray:
    y = np.ascontiguousarray(y, np.float32)
    out = np.empty(y.shape, np.float64)
    _chk(_load().orc_llr_biawgn(_p(y, _f32p), y.size, float(sigma2), float(llr_max), _p(out, _f64p)),
         "llr_biawgn")
    return out


def bp_decode(code, llr: np.ndarray, synd: np.ndarray, max_iter: int = 100, q_max: float = 40.0):
    """-> (bits uint32[F][ceil(n/32)], converged uint8[F], iters int32[F])."""
    llr = np.ascontiguousarray(llr, np.float64).reshape(-1, code.n)
    F = llr.shape[0]
    synd = np.ascontiguousarray(synd, np.uint32).reshape(F, words(code.m_checks))
    bits = np.empty((F, words(code.n)), np.uint32)
    conv = np.empty(F, np.uint8)
    iters = np.empty(F, np.int32)
    _chk(_load().orc_bp_decode(code.n, code.m_checks, _p(code.row_ptr, _i32p), _p(code.col_idx, _i32p),
                               _p(llr, _f64p), _p(synd, _u32p), F, max_iter, float(q_max),
                               _p(bits, _u32p), _p(conv, _u8p), _p(iters, _i32p)), "bp_decode")
    return bits, conv, iters


def layers(code) -> np.ndarray:
    """Greedy check colouring of the row-layered schedule (reading R-9): int32[M] layer per check."""
    out = np.empty(code.m_checks, np.int32)
    rc = _load().orc_layers(code.n, code.m_checks, _p(code.row_ptr, _i32p), _p(code.col_idx, _i32p),
                            _p(out, _i32p))
    if rc <= 0:
        raise RuntimeError(f"oracle layers failed ({rc})")
    return out


def bp_decode_layered(code, llr: np.ndarray, synd: np.ndarray, max_iter: int = 100, q_max: float = 40.0,
                      stop_early: bool = True, want_r: bool = False):
    """Row-layered sum-product (reading R-9).  -> (bits, converged, iters, post float64[F][n])
    (+ r float64[F][E], the check-to-variable messages in CSR edge order, if want_r)."""
    llr = np.ascontiguousarray(llr, np.float64).reshape(-1, code.n)
    F = llr.shape[0]
    synd = np.ascontiguousarray(synd, np.uint32).reshape(F, words(code.m_checks))
    bits = np.empty((F, words(code.n)), np.uint32)
    conv = np.empty(F, np.uint8)
    iters = np.empty(F, np.int32)
    post = np.empty((F, code.n), np.float64)
    r = np.empty((F, code.n_edges), np.float64) if want_r else None
    _chk(_load().orc_bp_layered(code.n, code.m_checks, _p(code.row_ptr, _i32p), _p(code.col_idx, _i32p),
                                _p(llr, _f64p), _p(synd, _u32p), F, max_iter, float(q_max), int(stop_early),
                                _p(bits, _u32p), _p(conv, _u8p), _p(iters, _i32p), _p(post, _f64p),
                                _p(r, _f64p) if want_r else None),
         "bp_layered")
    return (bits, conv, iters, post, r) if want_r else (bits, conv, iters, post)


def bp_trace_layered(code, llr: np.ndarray, synd: np.ndarray, k_iters: int, q_max: float = 40.0):
    """Row-layered schedule after exactly k iterations: -> (r float64[F][E] CSR order, post float64[F][n])."""
    _, _, _, post, r = bp_decode_layered(code, llr, synd, k_iters, q_max, stop_early=False, want_r=True)
    return r, post


def bp_trace(code, llr: np.ndarray, synd: np.ndarray, k_iters: int, q_max: float = 40.0):
    """-> (c2v float64[F][E] in CSR edge order, post float64[F][n]) after exactly k iterations."""
    llr = np.ascontiguousarray(llr, np.float64).reshape(-1, code.n)
    F = llr.shape[0]
    synd = np.ascontiguousarray(synd, np.uint32).reshape(F, words(code.m_checks))
    c2v = np.empty((F, code.n_edges), np.float64)
    post = np.empty((F, code.n), np.float64)
    _chk(_load().orc_bp_trace(code.n, code.m_checks, _p(code.row_ptr, _i32p), _p(code.col_idx, _i32p),
                              _p(llr, _f64p), _p(synd, _u32p), F, k_iters, float(q_max),
                              _p(c2v, _f64p), _p(post, _f64p)), "bp_trace")
    return c2v, post


SCHEDULES = {"flooding": 0, "layered": 1}


def reconcile(codes: Sequence, order: Sequence[int], edges: np.ndarray, sigma_n: float,
              x: np.ndarray, synd: Sequence[np.ndarray], max_iter: int = 100,
              q_max: float = 40.0, llr_max: float = 40.0, schedule: str = "flooding"):
    """Multi-stage driver O6.  codes[j] None => disclosed, synd[j] = Bob's packed bits.
    schedule: "flooding" (O5, reading A-8) or "layered" (O5', reading R-9) BP for the coded slices.

    -> (label uint8[F][n], frame_ok uint8[F], iters int32[F][m])."""
    m = len(codes)
    edges = np.ascontiguousarray(edges, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    F, n = x.shape
    nch = np.array([c.m_checks if c is not None else 0 for c in codes], np.int32)
    rp = (_i32p * m)(*[(_p(c.row_ptr, _i32p) if c is not None else _i32p()) for c in codes])
    ci = (_i32p * m)(*[(_p(c.col_idx, _i32p) if c is not None else _i32p()) for c in codes])
    synd = [np.ascontiguousarray(s, np.uint32) for s in synd]
    sp = (_u32p * m)(*[_p(s, _u32p) for s in synd])
    order = np.ascontiguousarray(order, np.int32)
    label = np.empty((F, n), np.uint8)
    ok = np.empty(F, np.uint8)
    iters = np.empty((F, m), np.int32)
    _chk(_load().orc_reconcile(m, n, _p(nch, _i32p), rp, ci, _p(order, _i32p), _p(edges, _f32p),
                               float(sigma_n), _p(x, _f32p), sp, F, max_iter, float(q_max),
                               float(llr_max), SCHEDULES[schedule], _p(label, _u8p), _p(ok, _u8p),
                               _p(iters, _i32p)),
         "reconcile")
    return label, ok, iters
