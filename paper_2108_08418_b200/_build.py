"""In-tree build of libcvsr.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libcvsr.so")
SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "cvsr.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for p in ("/usr/local/cuda/bin/nvcc",):
        if os.path.exists(p):
            return p
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile every .cu to an object in parallel, then link libcvsr.so (or `out`,
    with extra -D `defines`, for A/B variants)."""
    if out is None and not force and not stale():
        return LIB
    target = out or LIB
    import concurrent.futures as cf
    import tempfile
    objdir = tempfile.mkdtemp(prefix="cvsr_build_")
    flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *flags, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c", src,
               "-o", obj]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "".join(r.stderr for _, r in results)
    for _, r in results:
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stderr[-6000:])
    tmp = target + f".tmp{os.getpid()}"
    link = subprocess.run([nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                           *[o for o, _ in results], "-o", tmp], capture_output=True, text=True)
    if link.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + link.stderr[-6000:])
    if verbose:
        print(log)
    if out is None:
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write(log)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
