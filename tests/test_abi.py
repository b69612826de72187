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


SUPPORTED = {(3, 0), (3, 1), (2, 2)}   # (dim, kernel) pairs include/dmk.h lists


class _Opt(ctypes.Structure):
    """dmk_options, declared here from include/dmk.h (independent of the binding)."""
    _fields_ = [("leaf_capacity", ctypes.c_int32), ("min_level", ctypes.c_int32),
                ("lam", ctypes.c_double), ("stream", ctypes.c_void_p),
                ("root", ctypes.POINTER(ctypes.c_double)), ("n_targets", ctypes.c_int64)]


@pytest.fixture(scope="module")
def raw(lib):
    """A CDLL instance of its own (the binding's instance keeps its argtypes)."""
    import paper_2308_00292_b200 as dmk
    L = ctypes.CDLL(dmk.LIB_PATH)
    L.dmk_last_error.restype = ctypes.c_char_p
    return L


def _raw_plan(lib, dim, kernel, eps, pts, opt):
    h = ctypes.c_void_p()
    lib.dmk_plan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                             ctypes.c_int, ctypes.POINTER(_Opt), ctypes.POINTER(ctypes.c_void_p)]
    rc = lib.dmk_plan(dim, kernel, eps, pts.shape[0], pts.ctypes.data, 1, ctypes.byref(opt), ctypes.byref(h))
    return rc, h


def test_kernel_matrix_matches_header(raw):
    """Every (dim, kernel) pair the header lists passes argument validation (on a box
    without a GPU it then fails with DMK_ERR_CUDA, never UNSUPPORTED); every other pair
    is DMK_ERR_UNSUPPORTED."""
    torch = pytest.importorskip("torch")
    gpu = torch.cuda.is_available()
    for dim in (1, 2, 3, 4):
        for kernel in (0, 1, 2, 3):
            pts = np.random.default_rng(0).uniform(0, 1, (64, max(dim, 1)))
            rc, h = _raw_plan(raw, dim, kernel, 1e-6, pts, _Opt(16, 0, 1.0, None, None, 0))
            if (dim, kernel) in SUPPORTED:
                assert rc == (0 if gpu else -3), (dim, kernel, rc, raw.dmk_last_error())
                if gpu:
                    assert raw.dmk_destroy(h) == 0
            else:
                assert rc == -2, (dim, kernel, rc)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,kernel,eps", [(3, 0, 1e-6), (3, 1, 1e-6), (2, 2, 1e-9), (3, 0, 1e-3), (3, 1, 1e-9)])
def test_every_kernel_through_raw_abi(raw, dim, kernel, eps):
    """Raw ctypes (no binding): dmk_plan + dmk_eval on host buffers + dmk_destroy for each
    kernel enum, against the oracle's fp64 direct sum (2 eps)."""
    import dmk_inputs
    from oracle import direct
    if dim == 2:
        x, q = dmk_inputs.circle2d(3000, seed=3)
        ref = direct.log2d(x, q)
    else:
        x, q = dmk_inputs.uniform(3000, seed=3)
        ref = direct.yukawa3d(x, q, 10.0) if kernel == 1 else direct.laplace3d(x, q)
    x = np.ascontiguousarray(x)
    rc, h = _raw_plan(raw, dim, kernel, eps, x, _Opt(40, 0, 10.0, None, None, 0))
    assert rc == 0, raw.dmk_last_error()
    u = np.zeros(x.shape[0])
    raw.dmk_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    raw.dmk_destroy.argtypes = [ctypes.c_void_p]
    assert raw.dmk_eval(h, q.ctypes.data, u.ctypes.data, 1) == 0, raw.dmk_last_error()
    assert raw.dmk_destroy(h) == 0
    assert direct.rel_l2(u, ref) <= 2 * eps
