"""The C-ABI boundary: the library loads (no GPU needed) and exports every function that
include/lmoe_cuda.h declares; the C++ drop-in header compiles and its consumer runs on the
GPU; the product package has no CPU fallback."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lmoe_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmoe_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2503_05447_b200 import _build
    _build.build()
    lib = ctypes.CDLL(_build.LIB)  # loads without a GPU
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    from paper_2503_05447_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"\.(sm_\d+[a-z]?)\.cubin", out))
    assert archs == {"sm_100a"}, archs


def test_sass_uses_tcgen05_and_tma():
    """tcgen05.mma -> UTC*MMA, TMA -> UTMALDG in the shipped SASS (B200_PROFILING.md)."""
    from paper_2503_05447_b200 import _build
    sass = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", sass)
    assert "UTMALDG" in sass
    assert "LDTM" in sass


def test_host_errors_before_device_work():
    """Argument validation mirrors the reference texts and needs no GPU."""
    import paper_2503_05447_b200._lib as L
    lib = L.lib()
    d = L.LsmDesc()
    d.instance, d.use_normalizer, d.chunk_size = 13, 1, 64
    rc = lib.lmoe_lsm_fwd(ctypes.byref(d), 1, 8, 1, 128, 1, *([None] * 11), None, 0, None)
    assert rc != 0
    assert lib.lmoe_last_error().decode() == "LsmSpec: normalizer unsupported for instance mamba2"
    d.use_normalizer, d.chunk_size = 0, 0
    rc = lib.lmoe_lsm_fwd(ctypes.byref(d), 1, 8, 1, 128, 1, *([None] * 11), None, 0, None)
    assert lib.lmoe_last_error().decode() == "lsm_forward_chunked: chunk_size must be >= 1"


@pytest.mark.gpu
def test_cpp_dropin_api_runs():
    from paper_2503_05447_b200 import _build
    _build.build()
    r = subprocess.run([_build.CPP_API_BIN], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
