"""Thin Python binding of the cvsr C ABI (include/cvsr.h) -- argument marshalling only.

Every function has the C entry point's name and forwards to libcvsr.so
(sm_100a).  Buffers are torch tensors on the context's device (their
data_ptr() is passed), or raw integer device pointers.  There is no
fallback: if libcvsr.so is missing or fails to load, importing this module
raises, and every status other than CVSR_OK raises :class:`CvsrError`.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# CVSR_LIB: load another build of the same library (tools/build_variant.py A/B runs)
LIB_PATH = os.environ.get("CVSR_LIB") or os.path.join(_PKG, "libcvsr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
_lib = ctypes.CDLL(LIB_PATH)

CVSR_OK, CVSR_EINVAL, CVSR_ESHAPE, CVSR_ENOMEM, CVSR_ECUDA, CVSR_ECODE = 0, -1, -2, -3, -4, -5
_NAMES = {0: "CVSR_OK", -1: "CVSR_EINVAL", -2: "CVSR_ESHAPE", -3: "CVSR_ENOMEM", -4: "CVSR_ECUDA",
          -5: "CVSR_ECODE"}


class CvsrError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn}: {_NAMES.get(status, status)}: {msg}")
        self.status = status


class cvsr_quantiser(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("edges", ctypes.c_float * 255)]


class cvsr_decode_opts(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("msg_clamp", ctypes.c_float), ("flags", ctypes.c_int32)]


class cvsr_stats(ctypes.Structure):
    _fields_ = [("frames", ctypes.c_int64), ("frames_ok", ctypes.c_int64), ("bits_reconciled", ctypes.c_int64),
                ("attempted", ctypes.c_int64 * 8), ("converged", ctypes.c_int64 * 8),
                ("iters_sum", ctypes.c_int64 * 8), ("edge_iters", ctypes.c_int64 * 8),
                ("alice_seconds", ctypes.c_double), ("schedule", ctypes.c_int32 * 8)]

    def as_dict(self, m: int) -> dict:
        return {"frames": self.frames, "frames_ok": self.frames_ok, "bits_reconciled": self.bits_reconciled,
                "attempted": list(self.attempted)[:m], "converged": list(self.converged)[:m],
                "iters_sum": list(self.iters_sum)[:m], "edge_iters": list(self.edge_iters)[:m],
                "alice_seconds": self.alice_seconds, "schedule": list(self.schedule)[:m]}


_vp = ctypes.c_void_p
_i32, _i64, _u32, _f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_float
_P = ctypes.POINTER

_SIGS = {
    "cvsr_last_error": ([], ctypes.c_char_p),
    "cvsr_abi_version": ([], _i32),
    "cvsr_ctx_create": ([_i32, _vp, _P(_vp)], _i32),
    "cvsr_ctx_set_stream": ([_vp, _vp], _i32),
    "cvsr_ctx_sync": ([_vp], _i32),
    "cvsr_ctx_launch_count": ([_vp], _i64),
    "cvsr_ctx_destroy": ([_vp], None),
    "cvsr_ctx_set_profiling": ([_vp, _i32], _i32),
    "cvsr_ctx_kernel_times": ([_vp, _P(ctypes.c_double), _P(_i64)], _i32),
    "cvsr_code_load": ([_vp, _i32, _i32, _P(_i32), _P(_i32), _P(_vp)], _i32),
    "cvsr_code_info": ([_vp, _P(_i32), _P(_i32), _P(_i64)], _i32),
    "cvsr_code_free": ([_vp], None),
    "cvsr_quantise": ([_vp, _P(cvsr_quantiser), _vp, _i64, _vp], _i32),
    "cvsr_slice_bits": ([_vp, _vp, _i32, _i32, _i32, _vp], _i32),
    "cvsr_syndrome": ([_vp, _vp, _vp, _i32, _i32, _vp], _i32),
    "cvsr_llr_slice": ([_vp, _P(cvsr_quantiser), _vp, _i32, _i32, _f32, _i32, _u32, _vp, _f32, _vp], _i32),
    "cvsr_llr_biawgn": ([_vp, _vp, _i64, _f32, _f32, _vp], _i32),
    "cvsr_decode": ([_vp, _vp, _vp, _vp, _i32, _P(cvsr_decode_opts), _vp, _vp, _vp], _i32),
    "cvsr_decode_trace": ([_vp, _vp, _vp, _vp, _i32, _i32, _f32, _i32, _vp, _vp], _i32),
    "cvsr_reconcile": ([_vp, _i32, _P(_vp), _P(_i32), _P(cvsr_quantiser), _f32, _vp, _P(_vp), _i32, _i32,
                        _P(cvsr_decode_opts), _vp, _vp, _vp, _P(cvsr_stats)], _i32),
    "cvsr_count_errors": ([_vp, _vp, _vp, _vp, _i32, _i32, _P(_i64)], _i32),
    "cvsr_frame_hash": ([_vp, _vp, _i32, _i32, ctypes.c_uint64, _vp], _i32),
    "cvsr_session_set_verify": ([_vp, _vp], _i32),
    "cvsr_session_run_host_stream": ([_vp, _i32, _vp, _vp, _vp, _vp], _i32),
    "cvsr_pa_plan_create": ([_vp, _i64, _i64, _vp, _P(_vp)], _i32),
    "cvsr_pa_plan_info": ([_vp, _P(_i64), _P(_i64), _P(_i64)], _i32),
    "cvsr_pa_hash": ([_vp, _vp, _i32, _vp, _vp], _i32),
    "cvsr_pa_plan_free": ([_vp], None),
    "cvsr_verify": ([_vp, _vp, _vp, _vp, _i32, _i32, _P(ctypes.c_uint64), _vp, _vp, _vp], _i32),
    "cvsr_session_create": ([_vp, _i32, _P(_vp), _P(_i32), _P(cvsr_quantiser), _f32, _i32, _i32,
                             _P(cvsr_decode_opts), _P(_vp)], _i32),
    "cvsr_session_run": ([_vp, _vp, _vp, _P(cvsr_stats)], _i32),
    "cvsr_session_run_host": ([_vp, _vp, _vp, _vp, _vp, _vp, _P(cvsr_stats)], _i32),
    "cvsr_session_buffers": ([_vp, _P(_vp), _P(_vp), _P(_vp), _P(_vp)], _i32),
    "cvsr_session_destroy": ([_vp], None),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _ptr(t) -> Optional[int]:
    """Device pointer of a tensor (or an int pointer, or None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _call(name: str, *args):
    st = getattr(_lib, name)(*args)
    if st != CVSR_OK:
        raise CvsrError(st, name, _lib.cvsr_last_error().decode(errors="replace"))
    return st


def cvsr_last_error() -> str:
    return _lib.cvsr_last_error().decode(errors="replace")


def cvsr_abi_version() -> int:
    return int(_lib.cvsr_abi_version())


# ---------------------------------------------------------------- context

def cvsr_ctx_create(device: int = 0, stream=None) -> int:
    """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None (legacy default)."""
    h = _vp()
    s = getattr(stream, "cuda_stream", stream)
    _call("cvsr_ctx_create", device, s, ctypes.byref(h))
    return h.value


def cvsr_ctx_set_stream(ctx: int, stream) -> None:
    _call("cvsr_ctx_set_stream", ctx, getattr(stream, "cuda_stream", stream))


def cvsr_ctx_sync(ctx: int) -> None:
    _call("cvsr_ctx_sync", ctx)


def cvsr_ctx_launch_count(ctx: int) -> int:
    return int(_lib.cvsr_ctx_launch_count(ctx))


def cvsr_ctx_destroy(ctx: int) -> None:
    _lib.cvsr_ctx_destroy(ctx)


KERNEL_CLASSES = ("cn", "vn", "init", "ctrl")


def cvsr_ctx_set_profiling(ctx: int, enable: bool) -> None:
    _call("cvsr_ctx_set_profiling", ctx, 1 if enable else 0)


def cvsr_ctx_kernel_times(ctx: int) -> dict:
    ms = (ctypes.c_double * 4)()
    cnt = (_i64 * 4)()
    _call("cvsr_ctx_kernel_times", ctx, ms, cnt)
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


# ---------------------------------------------------------------- code

def cvsr_code_load(ctx: int, n_vars: int, n_checks: int, row_ptr: np.ndarray, col_idx: np.ndarray) -> int:
    rp = np.ascontiguousarray(row_ptr, np.int32)
    ci = np.ascontiguousarray(col_idx, np.int32)
    if len(rp) != n_checks + 1:
        raise ValueError("row_ptr must have n_checks + 1 entries")
    h = _vp()
    _call("cvsr_code_load", ctx, n_vars, n_checks, rp.ctypes.data_as(_P(_i32)), ci.ctypes.data_as(_P(_i32)),
          ctypes.byref(h))
    return h.value


def cvsr_code_info(code: int):
    n, m, e = _i32(), _i32(), _i64()
    _call("cvsr_code_info", code, ctypes.byref(n), ctypes.byref(m), ctypes.byref(e))
    return n.value, m.value, e.value


def cvsr_code_free(code: int) -> None:
    _lib.cvsr_code_free(code)


# ---------------------------------------------------------------- Bob

def make_quantiser(edges: np.ndarray) -> cvsr_quantiser:
    e = np.ascontiguousarray(edges, np.float32)
    m = int(round(np.log2(len(e) + 1)))
    if (1 << m) - 1 != len(e):
        raise ValueError("edge table must have 2^m - 1 entries")
    q = cvsr_quantiser()
    q.m = m
    ctypes.memmove(q.edges, e.ctypes.data, e.nbytes)
    return q


def cvsr_quantise(ctx: int, q: cvsr_quantiser, y, count: int, label_out) -> None:
    _call("cvsr_quantise", ctx, ctypes.byref(q), _ptr(y), count, _ptr(label_out))


def cvsr_slice_bits(ctx: int, label, frames: int, n: int, slice_j: int, bits_out) -> None:
    _call("cvsr_slice_bits", ctx, _ptr(label), frames, n, slice_j, _ptr(bits_out))


def cvsr_syndrome(ctx: int, code: int, label, frames: int, slice_j: int, synd_out) -> None:
    _call("cvsr_syndrome", ctx, code, _ptr(label), frames, slice_j, _ptr(synd_out))


# ---------------------------------------------------------------- Alice

def cvsr_llr_slice(ctx: int, q: cvsr_quantiser, x, frames: int, n: int, sigma_n: float, slice_j: int,
                   known_mask: int, known_label, llr_max: float, llr_out) -> None:
    _call("cvsr_llr_slice", ctx, ctypes.byref(q), _ptr(x), frames, n, sigma_n, slice_j, known_mask,
          _ptr(known_label), llr_max, _ptr(llr_out))


def cvsr_llr_biawgn(ctx: int, y, count: int, sigma2: float, llr_max: float, llr_out) -> None:
    _call("cvsr_llr_biawgn", ctx, _ptr(y), count, sigma2, llr_max, _ptr(llr_out))


CVSR_SCHED_DEFAULT, CVSR_SCHED_FLOODING, CVSR_SCHED_LAYERED = 0, 1, 2
SCHED = {"default": CVSR_SCHED_DEFAULT, "flooding": CVSR_SCHED_FLOODING, "layered": CVSR_SCHED_LAYERED}


def decode_opts(max_iter: int = 100, msg_clamp: float = 40.0, flags: int = 0) -> cvsr_decode_opts:
    """flags: CVSR_SCHED_* (an int, or a schedule name "flooding" / "layered" / "default")."""
    if isinstance(flags, str):
        flags = SCHED[flags]
    return cvsr_decode_opts(max_iter, msg_clamp, flags)


def cvsr_decode(ctx: int, code: int, llr, synd, frames: int, opts: cvsr_decode_opts, bits_out, converged_out,
                iters_out) -> None:
    _call("cvsr_decode", ctx, code, _ptr(llr), _ptr(synd), frames, ctypes.byref(opts), _ptr(bits_out),
          _ptr(converged_out), _ptr(iters_out))


def cvsr_decode_trace(ctx: int, code: int, llr, synd, frames: int, k_iters: int, msg_clamp: float, c2v_out,
                      post_out, flags=CVSR_SCHED_FLOODING) -> None:
    if isinstance(flags, str):
        flags = SCHED[flags]
    _call("cvsr_decode_trace", ctx, code, _ptr(llr), _ptr(synd), frames, k_iters, msg_clamp, flags, _ptr(c2v_out),
          _ptr(post_out))


def cvsr_reconcile(ctx: int, m: int, codes: Sequence[Optional[int]], order: Sequence[int], q: cvsr_quantiser,
                   sigma_n: float, x, synd: Sequence, frames: int, n: int, opts: cvsr_decode_opts, label_out,
                   frame_ok, iters, want_stats: bool = True) -> Optional[dict]:
    code_arr = (_vp * m)(*[c if c else None for c in codes])
    order_arr = (_i32 * m)(*order)
    synd_arr = (_vp * m)(*[_ptr(s) for s in synd])
    st = cvsr_stats() if want_stats else None
    _call("cvsr_reconcile", ctx, m, code_arr, order_arr, ctypes.byref(q), sigma_n, _ptr(x), synd_arr, frames, n,
          ctypes.byref(opts), _ptr(label_out), _ptr(frame_ok), _ptr(iters),
          ctypes.byref(st) if st is not None else None)
    return st.as_dict(m) if st is not None else None


def cvsr_frame_hash(ctx: int, label, frames: int, n: int, key: int, hash_out) -> None:
    _call("cvsr_frame_hash", ctx, _ptr(label), frames, n, key, _ptr(hash_out))


def cvsr_session_run_host_stream(sess: int, x_hosts, y_hosts, label_hosts, frame_ok_hosts) -> None:
    """Lists of host buffers, one per batch (torch CPU tensors, pinned, or numpy arrays);
    label_hosts entries may be None."""
    def hp(a):
        if a is None:
            return None
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
    nb = len(x_hosts)
    arr = lambda lst: (ctypes.c_void_p * max(1, nb))(*[hp(a) for a in lst])  # noqa: E731
    _call("cvsr_session_run_host_stream", sess, nb, arr(x_hosts), arr(y_hosts), arr(label_hosts),
          arr(frame_ok_hosts))


def cvsr_pa_plan_create(ctx: int, n_in: int, n_out: int, seed_bits) -> int:
    """seed_bits: host uint32 words (numpy), n_in + n_out - 1 bits LSB first."""
    import numpy as np
    seed = np.ascontiguousarray(seed_bits, dtype=np.uint32)
    if seed.size * 32 < n_in + n_out - 1:
        raise ValueError("seed too short")
    out = ctypes.c_void_p()
    _call("cvsr_pa_plan_create", ctx, n_in, n_out, seed.ctypes.data, ctypes.byref(out))
    return out.value


def cvsr_pa_plan_info(plan: int):
    a, b, c = _i64(), _i64(), _i64()
    _call("cvsr_pa_plan_info", plan, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return a.value, b.value, c.value


def cvsr_pa_hash(ctx: int, plan: int, blocks: int, x_bits, y_bits) -> None:
    _call("cvsr_pa_hash", ctx, plan, blocks, _ptr(x_bits), _ptr(y_bits))


def cvsr_pa_plan_free(plan: int) -> None:
    _lib.cvsr_pa_plan_free(plan)


CVSR_HASH_KEYS = 3


def _keys(keys):
    keys = list(keys)
    if len(keys) != CVSR_HASH_KEYS:
        raise ValueError(f"{CVSR_HASH_KEYS} keys expected")
    return (ctypes.c_uint64 * CVSR_HASH_KEYS)(*keys)


def cvsr_session_set_verify(sess: int, keys) -> None:
    """keys: CVSR_HASH_KEYS ints in [1, 2^61 - 2], or None (off)."""
    _call("cvsr_session_set_verify", sess, ctypes.cast(_keys(keys), _vp) if keys is not None else None)


def cvsr_verify(ctx: int, label_alice, label_bob, frame_ok, frames: int, n: int, keys, verified_out,
                hash_alice_out=None, hash_bob_out=None) -> None:
    """keys: CVSR_HASH_KEYS ints; hash outputs uint64[frames][CVSR_HASH_KEYS] (optional)."""
    _call("cvsr_verify", ctx, _ptr(label_alice), _ptr(label_bob), _ptr(frame_ok), frames, n, _keys(keys),
          _ptr(verified_out), _ptr(hash_alice_out) if hash_alice_out is not None else None,
          _ptr(hash_bob_out) if hash_bob_out is not None else None)


def cvsr_count_errors(ctx: int, label_alice, label_bob, frame_ok, frames: int, n: int):
    out = (_i64 * 3)()
    _call("cvsr_count_errors", ctx, _ptr(label_alice), _ptr(label_bob), _ptr(frame_ok), frames, n, out)
    return tuple(int(v) for v in out)


# ---------------------------------------------------------------- session

def cvsr_session_create(ctx: int, m: int, codes: Sequence[Optional[int]], order: Sequence[int], q: cvsr_quantiser,
                        sigma_n: float, n: int, frames: int, opts: cvsr_decode_opts) -> int:
    h = _vp()
    _call("cvsr_session_create", ctx, m, (_vp * m)(*[c if c else None for c in codes]), (_i32 * m)(*order),
          ctypes.byref(q), sigma_n, n, frames, ctypes.byref(opts), ctypes.byref(h))
    return h.value


def cvsr_session_run(sess: int, x, y, want_stats: bool = False, m: int = 8) -> Optional[dict]:
    st = cvsr_stats() if want_stats else None
    _call("cvsr_session_run", sess, _ptr(x), _ptr(y), ctypes.byref(st) if st is not None else None)
    return st.as_dict(m) if st is not None else None


def cvsr_session_run_host(sess: int, x_host, y_host, label_host, frame_ok_host, iters_host=None,
                          want_stats: bool = False, m: int = 8) -> Optional[dict]:
    """Host buffers: torch CPU tensors (pinned for overlapped copies) or numpy arrays."""
    def hp(a):
        if a is None:
            return None
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
    st = cvsr_stats() if want_stats else None
    _call("cvsr_session_run_host", sess, hp(x_host), hp(y_host), hp(label_host), hp(frame_ok_host), hp(iters_host),
          ctypes.byref(st) if st is not None else None)
    return st.as_dict(m) if st is not None else None


def cvsr_session_buffers(sess: int):
    a, b, c, d = _vp(), _vp(), _vp(), _vp()
    _call("cvsr_session_buffers", sess, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d))
    return a.value, b.value, c.value, d.value


def cvsr_session_destroy(sess: int) -> None:
    _lib.cvsr_session_destroy(sess)
