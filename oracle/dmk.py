"""The discrete DMK algorithm for the 3D Laplace and Yukawa kernels and the 2D log
kernel  (oracle; test infrastructure).

Follows "The full DMK algorithm for discrete sources", Sec. 3.5, PAPER.md:1414-1623,
step by step and in the paper's order, with the PSWF kernel split of Sec. 3.6
(oracle/kernels.py) and the Table 1 parameters (oracle/params.py):

  Step 0  tree + flags
  Step 1  precomputation of T_c2p, T_p2c, T_prox2pw, T_pw2poly,
          T_pwshift (1D factors)
  Step 2  upward pass: leaf proxy charges (Eq. 2.8), then c2p
  Step 3  downward pass per level: outgoing Phi_l (Eq. 3.42),
          incoming Psi_l (Eq. 3.39), local Lambda_l (Eqs. 3.43-3.44),
          split to children (T_p2c, Eq. 3.46), evaluate at
          leaf targets
  Step 4  direct residual interactions over the lists
  Step 5  self-interaction corrections

Kernels: 1/r with the PSWF split of Sec. 3.6 (LaplaceSplit), exp(-lam r)/r with the
Fourier-space PSWF split of Sec. 4.6, Eq. 4.18 (YukawaSplit), -log r in 2D with the same
split at lam = 0 (LogSplit2D).  The points are mapped to the unit
root box (x -> (x - lo)/side); the kernel there is K(side r'):
  3D: exp(-(lam side) r')/(side r')  -> run with lam' = lam side, divide by side;
  2D: -log r' - log side            -> subtract log(side) sum_{j: x_j != x_i} rho_j.
The algorithm is written for general d (Sec. 3.5 states it so): 2^d children, 3^d
colleagues, p^d Chebyshev tensors, (2 n_f + 1)^d plane waves.

Readings: R2 Fourier spacing, R4 root window M_1 = W_0 + D_0,
R5-R8 tree conventions, R9 coincident pairs, R10 root-leaf case (N <= n_s: plain
direct sum).  No blocking, fusion or reordering beyond the paper's; 1D factor
matrices are applied axis by axis (separation of variables, which the paper's
Step 1 prescribes).  Sources = targets; the potential at a source excludes the
source itself.
"""
from __future__ import annotations

import numpy as np

from . import cheb
from .kernels import LaplaceSplit, LogSplit2D, YukawaSplit, r_level, trapezoid_weights
from .params import for_eps
from .tree import Tree


def _octant_sides(code: int, d: int = 3):
    """Child orthant -> side (+-1) per axis; bit d-1-k of the child index is axis k."""
    o = int(code) & (2 ** d - 1)
    return [1 if (o >> (d - 1 - k)) & 1 else -1 for k in range(d)]


def dmk_laplace3d(points, charges, eps: float, ns: int, return_stages: bool = False):
    """u_i = sum_{j != i} rho_j / |x_i - x_j| by DMK.  points (N,3), charges (N,)."""
    return dmk(points, charges, eps, ns, "laplace", 0.0, return_stages)


def dmk_yukawa3d(points, charges, eps: float, ns: int, lam: float, return_stages: bool = False):
    """u_i = sum_{j != i} rho_j exp(-lam |x_i - x_j|)/|x_i - x_j| by DMK."""
    return dmk(points, charges, eps, ns, "yukawa", lam, return_stages)


def dmk_log2d(points, charges, eps: float, ns: int, return_stages: bool = False):
    """u_i = -sum_{j: x_j != x_i} rho_j log|x_i - x_j| by DMK.  points (N,2)."""
    return dmk(points, charges, eps, ns, "log", 0.0, return_stages)


def dmk3d(points, charges, eps, ns, kernel="laplace", lam=0.0, return_stages=False):
    return dmk(points, charges, eps, ns, kernel, lam, return_stages)


def _finish(T, us, rho, kernel, coinc_sum):
    """Back from the unit root box to the caller's units and order."""
    u = np.empty(T.N)
    if kernel == "log":
        u[T.perm] = us - np.log(T.side) * (np.sum(rho) - coinc_sum)
    else:
        u[T.perm] = us / T.side
    return u


def dmk(points, charges, eps: float, ns: int, kernel: str = "laplace", lam: float = 0.0,
        return_stages: bool = False, root=None, min_level: int = 0, level_get=None, level_set=None,
        box_get=None, box_set=None):
    """level_get = C: stop after Step 2 and return the proxy charges of every box of level
    C as a dense array [2^{dC}][p]*d indexed by Morton code (0 for absent boxes).
    level_set = (C, dense): after Step 2 replace the proxy charges of level C by `dense`
    and rebuild the coarser levels by T_c2p.  box_get = (C, codes): stop after Step 2 and
    return the proxy charges of the listed boxes of level C ([len(codes)][p]*d);
    box_set = [(C, codes, values), ...]: after Step 2 replace the proxy charges of the
    listed boxes (no rebuild), applied before level_set.  All need C < min_level; together
    with root/min_level they are the hooks of a distributed evaluation (they only move
    data: every value set is this function's own Step 2 output on some rank)."""
    T = Tree(points, ns, root=root, min_level=min_level)   # Step 0
    D = T.d
    prm = for_eps(eps, D)
    if kernel == "laplace" and D == 3:
        split = LaplaceSplit(prm.c)
        K = lambda r: 1.0 / r
    elif kernel == "yukawa" and D == 3:
        split = YukawaSplit(prm.c, lam * T.side)
        K = split.K
    elif kernel == "log" and D == 2:
        split = LogSplit2D(prm.c)
        K = split.K
    else:
        raise ValueError(f"kernel {kernel} in {D}D")
    rho = np.asarray(charges, dtype=np.float64)[T.perm]
    X = T.xs
    N = T.N
    st = {"tree": T, "params": prm, "split": split}
    if T.box_leaf[0]:                                      # reading R10: root is a leaf
        dx = X[:, None, :] - X[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", dx, dx))
        with np.errstate(divide="ignore"):
            inv = np.where(r > 0.0, K(np.where(r > 0.0, r, 1.0)), 0.0)
        us = inv @ rho
        coinc_sum = (r == 0.0) @ rho
        st.update(u_far=np.zeros(N), u_near=us, u_self=np.zeros(N))
        u = _finish(T, us, rho, kernel, coinc_sum)
        return (u, st) if return_stages else u

    p = prm.p
    # ---- Step 1: precomputation -------------------------------------------
    xn = cheb.nodes(p)
    Vi = cheb.Vinv(p)
    C2P = {s: cheb.c2p_1d(p, s) for s in (-1, 1)}
    P2C = {s: cheb.p2c_1d(p, s) for s in (-1, 1)}
    lev = {}
    for l in range(T.nlevels):
        h, nf = prm.h(l), prm.nfl(l)
        if l == 0:
            w = trapezoid_weights(lambda k: split.What_root(k, prm.RT), h, nf, D)
        else:
            w = trapezoid_weights(lambda k, l=l: split.Dhat(l, k), h, nf, D)
        m = np.arange(-nf, nf + 1, dtype=np.float64)
        s = r_level(l)
        E_out = np.exp(-1j * h * np.outer(m, xn * s / 2.0))     # T_prox2pw 1D factor (N1, p)
        E_in = np.exp(1j * h * np.outer(xn * s / 2.0, m))       # T_pw2poly 1D factor (p, N1)
        shift = {dd: np.exp(1j * h * m * dd * s) for dd in (-1, 0, 1)}   # T_pwshift factors
        lev[l] = dict(h=h, nf=nf, w=w, E_out=E_out, E_in=E_in, shift=shift)

    def outer_shift(L, dd):
        out = L["shift"][dd[0]]
        for k in range(1, D):
            out = np.multiply.outer(out, L["shift"][dd[k]])
        return out

    # ---- Step 2: upward pass -----------------------------------------------
    proxy = {}
    for i in np.nonzero(T.box_leaf & (T.box_npts > 0))[0]:
        a, b = T.box_start[i], T.box_end[i]
        c, s = T.center(i), r_level(T.box_level[i])
        U = [cheb.interp_matrix(2.0 * (X[a:b, k] - c[k]) / s, p) for k in range(D)]
        spec = ",".join("j" + "abc"[k] for k in range(D)) + ",j->" + "abc"[:D]
        proxy[i] = np.einsum(spec, *U, rho[a:b], optimize=True)
    def c2p_levels(top):
        for l in range(top, -1, -1):
            for i in range(T.level_offset[l], T.level_offset[l + 1]):
                if not T.fout[i]:
                    continue
                acc = np.zeros((p,) * D)
                for ch in T.box_children[i]:
                    if ch >= 0 and ch in proxy:
                        sd = _octant_sides(T.box_code[ch], D)
                        acc += cheb.applyd([C2P[sd[k]] for k in range(D)], proxy[ch])
                proxy[i] = acc

    c2p_levels(T.nlevels - 2)

    def box_index(C):
        return {int(T.box_code[i]): i for i in range(T.level_offset[C], T.level_offset[C + 1])}

    if box_get is not None:
        C, codes = int(box_get[0]), box_get[1]
        ix = box_index(C)
        out = np.zeros((len(codes),) + (p,) * D)
        for k, c in enumerate(codes):
            i = ix.get(int(c))
            if i is not None and i in proxy:
                out[k] = proxy[i]
        return out
    for C, codes, vals in (box_set or []):
        ix = box_index(int(C))
        for c, v in zip(codes, vals):
            i = ix.get(int(c))
            if i is not None and T.fout[i]:
                proxy[i] = np.array(v)
    if level_get is not None:
        C = int(level_get)
        dense = np.zeros((2 ** (D * C),) + (p,) * D)
        for i in range(T.level_offset[C], T.level_offset[C + 1]):
            if i in proxy:
                dense[T.box_code[i]] = proxy[i]
        return dense
    if level_set is not None:
        C, dense = int(level_set[0]), level_set[1]
        for i in range(T.level_offset[C], T.level_offset[C + 1]):
            if T.fout[i]:
                proxy[i] = np.array(dense[T.box_code[i]])
        c2p_levels(C - 1)
    st["proxy"] = proxy

    # ---- Step 3: downward pass ---------------------------------------------
    Phi, Psi, local = {}, {}, {}
    u_far = np.zeros(N)
    for l in range(T.nlevels):
        L = lev[l]
        rng_ = range(T.level_offset[l], T.level_offset[l + 1])
        for i in rng_:                                    # outgoing expansions
            if T.fout[i]:
                Phi[i] = cheb.applyd([L["E_out"]] * D, proxy[i])
        for i in rng_:                                    # incoming expansions
            if T.fin[i]:
                acc = np.zeros_like(L["w"], dtype=np.complex128)
                for sb in T.pwlist[i]:
                    dd = T.box_coords[i] - T.box_coords[sb]
                    acc += L["w"] * outer_shift(L, dd) * Phi[sb]
                Psi[i] = acc
        for i in rng_:                                    # local expansions
            if T.box_npts[i] == 0:
                continue
            lam_ = np.zeros((p,) * D)
            if T.fin[i]:
                vals = cheb.applyd([L["E_in"]] * D, Psi[i]).real
                lam_ += cheb.applyd([Vi] * D, vals)
            par = T.box_parent[i]                         # split from parent (Eq. 3.46)
            if par >= 0 and par in local:
                sd = _octant_sides(T.box_code[i], D)
                lam_ += cheb.applyd([P2C[sd[k]] for k in range(D)], local[par])
            local[i] = lam_
        for i in rng_:                                    # evaluate at leaf targets
            if T.box_leaf[i] and T.box_npts[i] > 0:
                a, b = T.box_start[i], T.box_end[i]
                c, s = T.center(i), r_level(l)
                E = [cheb.vander(2.0 * (X[a:b, k] - c[k]) / s, p) for k in range(D)]
                spec = ",".join("j" + "abc"[k] for k in range(D)) + "," + "abc"[:D] + "->j"
                u_far[a:b] = np.einsum(spec, *E, local[i], optimize=True)
    st.update(Phi=Phi, Psi=Psi, local=local)

    # ---- Step 4: direct interactions (residual kernel of the SOURCE level) ----
    u_near = np.zeros(N)
    for i in np.nonzero(T.box_leaf & (T.box_npts > 0))[0]:
        a, b = T.box_start[i], T.box_end[i]
        for sb in T.dlist[i]:
            sa, se = T.box_start[sb], T.box_end[sb]
            dx = X[a:b, None, :] - X[None, sa:se, :]
            r = np.sqrt(np.einsum("ijk,ijk->ij", dx, dx))
            R = np.where(r > 0.0, split.R(int(T.box_level[sb]), np.where(r > 0, r, 1.0)), 0.0)
            u_near[a:b] += R @ rho[sa:se]

    # ---- Step 5: self-interaction corrections --------------------------------
    u_self = np.zeros(N)
    coinc_sum = np.zeros(N)
    for i in np.nonzero(T.box_leaf & (T.box_npts > 0))[0]:
        a, b = T.box_start[i], T.box_end[i]
        dx = X[a:b, None, :] - X[None, a:b, :]
        coinc = np.all(dx == 0.0, axis=2)
        coinc_sum[a:b] = coinc @ rho[a:b]
        u_self[a:b] -= split.M0_at_zero(int(T.box_level[i])) * coinc_sum[a:b]

    us = u_far + u_near + u_self
    st.update(u_far=u_far, u_near=u_near, u_self=u_self)
    u = _finish(T, us, rho, kernel, coinc_sum)
    return (u, st) if return_stages else u
