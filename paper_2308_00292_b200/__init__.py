"""paper_2308_00292_b200 -- B200-native DMK (arXiv 2308.00292) for 3D Laplace.

Thin ctypes binding over the C ABI in ``include/dmk.h`` (libdmk.so, built in-tree
for sm_100a by ``paper_2308_00292_b200/build.py``).  Argument marshalling only:
every step of the computation runs in the library's CUDA kernels.  There is no
CPU path -- if the library or a CUDA device is missing, calls raise.

    plan = dmk_plan(points, eps=1e-6, leaf_capacity=200)   # torch.cuda (n,3) f64 or numpy (n,3)
    u = plan.eval(charges)                                  # same placement as `charges`
    plan.close()

Function names mirror the C entry points (dmk_plan, dmk_eval, dmk_destroy,
dmk_plan_info_get, dmk_tree_copy, dmk_stage_copy).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DMK_LIB") or os.path.join(_HERE, "libdmk.so")

DMK_OK = 0
DMK_MEM_DEVICE, DMK_MEM_HOST = 0, 1
DMK_KERNEL_LAPLACE, DMK_KERNEL_YUKAWA, DMK_KERNEL_LOG = 0, 1, 2
KERNELS = {"laplace": DMK_KERNEL_LAPLACE, "yukawa": DMK_KERNEL_YUKAWA, "log": DMK_KERNEL_LOG}
TREE = {name: i for i, name in enumerate(
    ["perm", "box_level", "box_code", "box_start", "box_end", "box_leaf", "box_parent",
     "colleagues", "dlist_off", "dlist", "fout", "exp"])}
STAGE = {"moments": 0, "outgoing": 1, "local": 2, "ufar": 3, "unear": 4}


class DmkError(RuntimeError):
    pass


class _Options(ctypes.Structure):
    _fields_ = [("leaf_capacity", ctypes.c_int32), ("min_level", ctypes.c_int32),
                ("lam", ctypes.c_double), ("stream", ctypes.c_void_p),
                ("root", ctypes.POINTER(ctypes.c_double)), ("n_targets", ctypes.c_int64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nbox", ctypes.c_int64), ("nlevels", ctypes.c_int32),
                ("p", ctypes.c_int32), ("nf", ctypes.c_int32), ("nf0", ctypes.c_int32),
                ("nfout", ctypes.c_int64), ("nexp", ctypes.c_int64), ("ndlist", ctypes.c_int64),
                ("lo", ctypes.c_double * 3), ("side", ctypes.c_double), ("c", ctypes.c_double),
                ("respoly_degree", ctypes.c_int32), ("dim", ctypes.c_int32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdmk.so (built in-tree); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DmkError(f"{LIB_PATH} not built; run __graft_entry__.build() or "
                           "python paper_2308_00292_b200/build.py")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.dmk_plan.argtypes = [ci, ci, dbl, i64, vp, ci, ctypes.POINTER(_Options), ctypes.POINTER(vp)]
        L.dmk_eval.argtypes = [vp, vp, vp, ci]
        L.dmk_upward.argtypes = [vp, vp, ci]
        L.dmk_downward.argtypes = [vp, vp, ci]
        L.dmk_level_moments.argtypes = [vp, ci, vp, i64, ci, ci]
        L.dmk_box_moments.argtypes = [vp, ci, vp, i64, vp, ci, ci]
        L.dmk_destroy.argtypes = [vp]
        L.dmk_last_error.restype = ctypes.c_char_p
        L.dmk_version.restype = ctypes.c_char_p
        L.dmk_plan_info_get.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        L.dmk_tree_copy.argtypes = [vp, ci, vp]
        L.dmk_stage_copy.argtypes = [vp, ci, vp, i64]
        L.dmk_stage_size.argtypes = [vp, ci]
        L.dmk_stage_size.restype = i64
        L.dmk_eval_timings.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(ctypes.c_char_p), ci]
        for f in ("dmk_plan", "dmk_eval", "dmk_upward", "dmk_downward", "dmk_level_moments", "dmk_box_moments",
                  "dmk_destroy", "dmk_plan_info_get", "dmk_tree_copy",
                  "dmk_stage_copy", "dmk_eval_timings"):
            getattr(L, f).restype = ci
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != DMK_OK:
        raise DmkError(f"{what} failed ({rc}): {lib().dmk_last_error().decode()}")


def _placement(a):
    """(pointer, mem, keepalive) for a torch tensor or numpy array of float64."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                raise DmkError("expected float64")
            a = a.contiguous()
            return a.data_ptr(), (DMK_MEM_DEVICE if a.is_cuda else DMK_MEM_HOST), a
    except ImportError:
        pass
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return arr.ctypes.data, DMK_MEM_HOST, arr


class Plan:
    """A dmk_plan_t: tree, lists and tables for one point set (sources = targets)."""

    def __init__(self, points, eps: float = 1e-6, leaf_capacity: int = 200, kernel: str = "laplace",
                 lam: float = 0.0, stream=None, root=None, min_level: int = 0, n_targets: int = 0):
        ptr, mem, keep = _placement(points)
        n = keep.shape[0]
        if keep.ndim != 2 or keep.shape[1] not in (2, 3):
            raise DmkError("points must have shape (n, 3) or (n, 2)")
        dim = int(keep.shape[1])
        self._root = None
        rootp = None
        if root is not None:
            self._root = (ctypes.c_double * (dim + 1))(*[float(v) for v in root])
            rootp = ctypes.cast(self._root, ctypes.POINTER(ctypes.c_double))
        opt = _Options(int(leaf_capacity), int(min_level), float(lam), stream, rootp, int(n_targets))
        h = ctypes.c_void_p()
        _check(lib().dmk_plan(dim, KERNELS[kernel], float(eps), int(n), ptr, mem, ctypes.byref(opt),
                              ctypes.byref(h)), "dmk_plan")
        self._h = h
        self.n = int(n)
        # the plan's stream may still read the points after dmk_plan returns (no
        # synchronisation there): keep them alive until close()
        self._points = keep

    def eval(self, charges, out=None):
        """Potentials u_i = sum_{j: x_j != x_i} K(|x_i - x_j|) rho_j (caller order)."""
        qptr, mem, qkeep = _placement(charges)
        if qkeep.shape != (self.n,):
            raise DmkError("charges must have shape (n,)")
        if out is None:
            if mem == DMK_MEM_DEVICE:
                import torch
                out = torch.empty(self.n, dtype=torch.float64, device=qkeep.device)
            else:
                out = np.empty(self.n, dtype=np.float64)
        optr, omem, okeep = _placement(out)
        if omem != mem:
            raise DmkError("charges and output must live in the same memory")
        _check(lib().dmk_eval(self._h, qptr, optr, mem), "dmk_eval")
        return okeep

    def upward(self, charges):
        """Step 2 only: moments of the charges (caller order), kept in the plan."""
        qptr, mem, qkeep = _placement(charges)
        if qkeep.shape != (self.n,):
            raise DmkError("charges must have shape (n,)")
        _check(lib().dmk_upward(self._h, qptr, mem), "dmk_upward")

    def downward(self, out=None, device=None):
        """Steps 3-5 from the plan's moments; returns the potentials (caller order)."""
        if out is None:
            if device is not None:
                import torch
                out = torch.empty(self.n, dtype=torch.float64, device=device)
            else:
                out = np.empty(self.n, dtype=np.float64)
        optr, mem, okeep = _placement(out)
        _check(lib().dmk_downward(self._h, optr, mem), "dmk_downward")
        return okeep

    def level_moments(self, level: int, dense=None, set: bool = False):
        """Dense [8^level, p, p, p] moments of the boxes at `level` (read, or write with
        set=True and rebuild the coarser levels)."""
        p = self.info().p
        if dense is None:
            dense = np.empty((8 ** level, p, p, p), dtype=np.float64)
        ptr, mem, keep = _placement(dense)
        _check(lib().dmk_level_moments(self._h, int(level), ptr, int(keep.numel() if hasattr(keep, "numel")
                                                                       else keep.size), mem, int(bool(set))),
               "dmk_level_moments")
        return keep

    def box_moments(self, level: int, codes, values=None, set: bool = False):
        """Moments [len(codes), p, p, p] of the listed boxes (Morton codes at `level`): read,
        or overwrite with set=True (no rebuild of other levels)."""
        p = self.info().p
        try:
            import torch
            dev_codes = isinstance(codes, torch.Tensor) and codes.is_cuda
        except ImportError:
            dev_codes = False
        if dev_codes:
            codes = codes.to(torch.int64).contiguous()
            cptr, nb = codes.data_ptr(), int(codes.numel())
        else:
            codes = np.ascontiguousarray(np.asarray(codes, dtype=np.int64))
            cptr, nb = codes.ctypes.data, int(codes.size)
        if values is None:
            values = np.empty((nb, p, p, p), dtype=np.float64)
        ptr, mem, keep = _placement(values)
        if (mem == DMK_MEM_DEVICE) != dev_codes:
            raise DmkError("codes and values must live in the same memory")
        _check(lib().dmk_box_moments(self._h, int(level), cptr, nb, ptr, mem, int(bool(set))), "dmk_box_moments")
        self._keep_codes = codes   # stream-ordered use of device codes
        return keep

    def info(self) -> PlanInfo:
        inf = PlanInfo()
        _check(lib().dmk_plan_info_get(self._h, ctypes.byref(inf)), "dmk_plan_info_get")
        return inf

    def tree(self, which: str) -> np.ndarray:
        inf = self.info()
        size = {"perm": inf.n, "colleagues": (9 if inf.dim == 2 else 27) * inf.nbox, "dlist_off": inf.nbox + 1,
                "dlist": inf.ndlist}.get(which, inf.nbox)
        out = np.empty(size, dtype=np.int64)
        _check(lib().dmk_tree_copy(self._h, TREE[which], out.ctypes.data), "dmk_tree_copy")
        return out

    def stage(self, which: str) -> np.ndarray:
        k = STAGE[which]
        size = int(lib().dmk_stage_size(self._h, k))
        out = np.empty(size, dtype=np.float64)
        _check(lib().dmk_stage_copy(self._h, k, out.ctypes.data, size), "dmk_stage_copy")
        return out

    def timings(self) -> dict:
        ms = (ctypes.c_double * 32)()
        names = (ctypes.c_char_p * 32)()
        k = lib().dmk_eval_timings(self._h, ms, names, 32)
        if k < 0:
            raise DmkError(f"dmk_eval_timings failed ({k}): {lib().dmk_last_error().decode()}")
        return {names[i].decode(): ms[i] for i in range(max(k, 0))}

    def close(self):
        if getattr(self, "_h", None):
            lib().dmk_destroy(self._h)
            self._h = None
        self._points = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def dmk_plan(points, eps: float = 1e-6, leaf_capacity: int = 200, kernel: str = "laplace", lam: float = 0.0,
             stream=None, root=None, min_level: int = 0, n_targets: int = 0) -> Plan:
    return Plan(points, eps=eps, leaf_capacity=leaf_capacity, kernel=kernel, lam=lam, stream=stream, root=root,
                min_level=min_level, n_targets=n_targets)


def dmk_eval(plan: Plan, charges, out=None):
    return plan.eval(charges, out)


def dmk_destroy(plan: Plan):
    plan.close()


def version() -> str:
    return lib().dmk_version().decode()
