"""C-ABI library: builds for sm_100a, loads, exports every symbol include/cvsr.h declares (CPU only)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "cvsr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cvsr_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2108_08418_b200 import _build
    path = _build.build()
    return ctypes.CDLL(path), path


def test_exports_every_declared_symbol(lib):
    L, path = lib
    names = _declared_symbols()
    assert len(names) >= 17
    for name in names:
        assert hasattr(L, name), name
    # and the binding wraps each of them under the same name
    from paper_2108_08418_b200 import cvsr
    assert set(names) == set(cvsr.EXPORTED)


def test_sass_is_sm100a(lib):
    _, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_error_paths_without_gpu(lib):
    from paper_2108_08418_b200 import cvsr
    assert cvsr.cvsr_abi_version() == 2
    with pytest.raises(cvsr.CvsrError) as ei:
        cvsr._call("cvsr_ctx_sync", None)
    assert ei.value.status == cvsr.CVSR_EINVAL
    assert "null context" in cvsr.cvsr_last_error()


def test_oracle_shares_no_code_with_cuda_path():
    """The oracle and the CUDA package never import/include each other."""
    for d, other in (("oracle", "paper_2108_08418_b200"), ("paper_2108_08418_b200", "oracle")):
        for dirpath, _, files in os.walk(os.path.join(ROOT, d)):
            for f in files:
                if f.endswith((".py", ".c", ".cu", ".cuh", ".h")):
                    txt = open(os.path.join(dirpath, f)).read()
                    assert not re.search(rf"^\s*(import|from)\s+{other}\b", txt, re.M), (f, other)
                    assert not re.search(rf'^\s*#\s*include\s*[<"][^>"]*{other}', txt, re.M), (f, other)
                    assert not re.search(rf"CDLL\([^)]*{other}", txt), (f, other)
