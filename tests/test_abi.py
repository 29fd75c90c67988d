"""CPU-side checks of the boundary: libscalegann.so builds, loads without a GPU and exports
every function include/scalegann.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "scalegann.h")).read()
    return sorted(set(re.findall(r"\b(scalegann_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_10135_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_the_header():
    from paper_2605_10135_b200 import api
    assert sorted(api.EXPORTS) == _declared()


def test_abi_version_and_error_plumbing(lib):
    lib.scalegann_abi_version.restype = ctypes.c_int
    assert lib.scalegann_abi_version() == 2
    lib.scalegann_last_error.restype = ctypes.c_char_p
    # argument validation happens before any CUDA call: a null pointer is rejected on the host
    lib.scalegann_prune.restype = ctypes.c_int
    st = lib.scalegann_prune(None, None, ctypes.c_uint64(10), 8, 4, 0, None, None, None)
    assert st == 1
    assert b"null" in lib.scalegann_last_error()


def test_validation_rejects_bad_degrees(lib):
    lib.scalegann_prune.restype = ctypes.c_int
    p = ctypes.c_void_p(16)
    assert lib.scalegann_prune(p, p, ctypes.c_uint64(10), 8, 9, 0, p, p, None) == 1      # R > L
    assert lib.scalegann_prune(p, p, ctypes.c_uint64(10), 300, 9, 0, p, p, None) == 1    # L > 256


def test_sass_has_tcgen05_and_tma(lib):
    """The distance kernel is tcgen05 + TMA code (UTC*MMA / UTMALDG in SASS)."""
    import subprocess
    from paper_2605_10135_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


def test_no_oracle_on_product_path():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2605_10135_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.c" not in txt, f
