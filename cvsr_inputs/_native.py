"""Build/load the host-only C construction library (input generator, no method arithmetic)."""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "ldpc_construct.c")
_LIB = os.path.join(_HERE, "libcvsr_inputs.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile libcvsr_inputs.so in-tree with gcc (no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i32p = ctypes.POINTER(ctypes.c_int32)
            L.ldpc_configuration_model.argtypes = [ctypes.c_int32, ctypes.c_int32, i32p, i32p,
                                                   ctypes.c_uint64, i32p, i32p]
            L.ldpc_configuration_model.restype = ctypes.c_int
            L.ldpc_permutation.argtypes = [ctypes.c_int32, ctypes.c_uint64, i32p]
            L.ldpc_permutation.restype = ctypes.c_int
            L.ldpc_peg.argtypes = [ctypes.c_int32, ctypes.c_int32, i32p, i32p, ctypes.c_uint64, ctypes.c_int32,
                                   i32p, i32p]
            L.ldpc_peg.restype = ctypes.c_int
            _lib = L
    return _lib
