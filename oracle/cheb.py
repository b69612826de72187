"""Chebyshev interpolation and anterpolation  (oracle; test infrastructure).

Sec. 2.1-2.2 of the paper.

    nodes of the first kind  r_i = cos(pi (i - 1/2)/p),  i = 1..p
    V(i,j) = T_{j-1}(r_i)
    E(k,n) = T_{n-1}(xi_k),  U = E V^{-1}  (interpolation)            PAPER.md:258-264, Eq. 2.1
    U^T = anterpolation; proxy charges rho~ = U^T rho                 Def. 2.1, Eqs. 2.4/2.8
    T_c2p = U^T with U from the parent grid to a child grid           Lemma 2.2
    T_p2c = V^{-1} E (coefficients, parent -> child)                  Lemma 2.3, Eq. 2.10

A box of side s centred at c maps x -> xi = 2 (x - c)/s in [-1,1].  A child of
that box (side s/2, centre c +- s/4) has xi_parent = xi_child/2 +- 1/2.
All 3D operators are tensor products of the 1D matrices below (separation of
variables).
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import chebyshev as npcheb


def nodes(p: int) -> np.ndarray:
    """First-kind Chebyshev nodes r_i, i = 1..p."""
    i = np.arange(1, p + 1, dtype=np.float64)
    return np.cos(np.pi * (i - 0.5) / p)


def vander(x, p: int) -> np.ndarray:
    """E(k, n) = T_{n-1}(x_k), shape (len(x), p)."""
    return npcheb.chebvander(np.asarray(x, dtype=np.float64), p - 1)


def V(p: int) -> np.ndarray:
    return vander(nodes(p), p)


def Vinv(p: int) -> np.ndarray:
    """V^{-1} by a library solve (numpy.linalg.inv)."""
    return np.linalg.inv(V(p))


def interp_matrix(x, p: int) -> np.ndarray:
    """U = E V^{-1}: node values -> values at points x (Eq. 2.1)."""
    return vander(x, p) @ Vinv(p)


def c2p_1d(p: int, side: int) -> np.ndarray:
    """1D factor of T_c2p for the child on side `side` (-1 or +1): the parent proxy
    charges from the child's proxy charges, i.e. the anterpolation U^T with U the
    interpolation from the parent grid to the child's nodes (Lemma 2.2)."""
    child_nodes_in_parent = nodes(p) / 2.0 + side * 0.5
    return interp_matrix(child_nodes_in_parent, p).T


def p2c_1d(p: int, side: int) -> np.ndarray:
    """1D factor of T_p2c = V^{-1} E (Lemma 2.3, Eq. 2.10): parent Chebyshev
    coefficients -> child Chebyshev coefficients.  E evaluates the parent basis at
    the child nodes."""
    child_nodes_in_parent = nodes(p) / 2.0 + side * 0.5
    return Vinv(p) @ vander(child_nodes_in_parent, p)


def apply3(mats, t):
    """Apply 1D matrices along the three axes of a (p,p,p)-like tensor:
    out[a,b,c] = sum_{ijk} M0[a,i] M1[b,j] M2[c,k] t[i,j,k]."""
    return np.einsum("ai,bj,ck,ijk->abc", mats[0], mats[1], mats[2], t, optimize=True)


def applyd(mats, t):
    """Apply 1D matrices along every axis of a d-dimensional tensor (d = len(mats))."""
    d = len(mats)
    ins = "ijk"[:d]
    outs = "abc"[:d]
    spec = ",".join(o + i for o, i in zip(outs, ins)) + "," + ins + "->" + outs
    return np.einsum(spec, *mats, t, optimize=True)
