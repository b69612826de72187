"""The C-ABI library loads, exports every symbol include/dmk.h declares, and fails
loudly (never falls back to the CPU) when arguments are bad or no GPU exists."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dmk.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dmk_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import paper_2308_00292_b200 as dmk
    if not os.path.exists(dmk.LIB_PATH):
        from paper_2308_00292_b200 import build
        build.build()
    return dmk.lib()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert "dmk_plan" in names and "dmk_eval" in names and len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name


def test_version_string(lib):
    assert b"sm_100a" in lib.dmk_version()


def test_bad_arguments_rejected(lib):
    import paper_2308_00292_b200 as dmk
    h = ctypes.c_void_p()
    pts = np.zeros((4, 3))
    # n = 0
    rc = lib.dmk_plan(3, 0, 1e-6, 0, pts.ctypes.data, 1, None, ctypes.byref(h))
    assert rc == -1 and b"n must be" in lib.dmk_last_error()
    # null points
    assert lib.dmk_plan(3, 0, 1e-6, 4, None, 1, None, ctypes.byref(h)) == -1
    # unsupported dimension / kernel
    assert lib.dmk_plan(2, 0, 1e-6, 4, pts.ctypes.data, 1, None, ctypes.byref(h)) == -2
    assert lib.dmk_plan(3, 2, 1e-6, 4, pts.ctypes.data, 1, None, ctypes.byref(h)) == -2   # log is 2D
    # Yukawa needs lambda > 0
    assert lib.dmk_plan(3, 1, 1e-6, 4, pts.ctypes.data, 1, None, ctypes.byref(h)) == -1
    assert b"lambda" in lib.dmk_last_error()
    # precision tighter than Table 1's 1e-9 row
    assert lib.dmk_plan(3, 0, 1e-12, 4, pts.ctypes.data, 1, None, ctypes.byref(h)) == -2
    # eval on a null plan
    assert lib.dmk_eval(None, pts.ctypes.data, pts.ctypes.data, 1) == -1
    with pytest.raises(dmk.DmkError):
        dmk.dmk_plan(np.zeros((0, 3)))


def test_no_cpu_fallback_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2308_00292_b200 as dmk
    with pytest.raises(dmk.DmkError, match="no CUDA device"):
        dmk.dmk_plan(np.random.default_rng(0).uniform(0, 1, (100, 3)))
