"""PSWF kernel splitting of the 3D Laplace kernel 1/r  (oracle; test infrastructure).

Paper: Sec. 3.6 "Optimization of kernel splitting using prolate spheroidal wave
functions".

    Phi_l(r) = (1/c0) int_0^{r/r_l} psi(x) dx
    W_0(r)   = Phi_0(r)/r,   D_l(r) = (Phi_{l+1}(r) - Phi_l(r))/r,
    R_L(r)   = (1 - Phi_L(r))/r                                Eq. 3.66
    1/r      = W_0 + sum_{l<L} D_l + R_L
    Dhat_l(k) = (4 pi/psi(0)) (psi(k r_{l+1}/c) - psi(k r_l/c)) / k^2,
    Dhat_l(0) = (2 pi c2/c0)(r_l^2 - r_{l+1}^2)                Eq. 3.68

with r_l = 2^{-l} the side of a level-l box.  We write
M_l(r) = Phi_l(r)/r for the mollified kernel at level l (Eq. 3.26 analogue,
PAPER.md:860-863), so D_l = M_{l+1} - M_l and R_L = 1/r - M_L.

Root level (reading R4 in DESIGN.md): the root box handles W_0 + D_0 = M_1 in one
Fourier sum.  Its Fourier transform is made smooth with the truncated-kernel
window of Sec. 4.7: Mhat_1(k) = Ghat_1(k) Khat(k) with
Ghat_1(k) = psi(k r_1/c)/psi(0), and the windowed kernel is
    What(k) = Ghat_1(k) That(k),  That(k) = 8 pi sin^2(k R_T/2)/k^2  (1/r truncated at R_T),
the PSWF analogue of Eq. 3.9 / Eq. 3.69.  With
R_T = (1 + sqrt 3) r_0 What equals M_1 for |x| <= sqrt 3.

Fourier discretisation (reading R2): trapezoidal rule with spacing h,
    f(x) ~= (h/2pi)^3 sum_m fhat(h m) e^{i h m.x}
(Eq. 3.35-3.37, with the h^3 quadrature weight the garbled
Eq. 3.35 omits).  Period 2pi/h must exceed the support diameter seen by the
sums: 3 r_l at level l >= 1, 1 + R_T + r_1 at the root.
"""
from __future__ import annotations

import numpy as np

from .pswf import Pswf


def r_level(l: int) -> float:
    """Box side at level l, r_l = 2^{-l}."""
    return 2.0 ** (-l)


class LaplaceSplit:
    """Kernel split of K(r) = 1/r for one PSWF parameter c."""

    def __init__(self, c: float):
        self.psi = Pswf(c)
        self.c = self.psi.c

    # ---- physical space -------------------------------------------------
    def M(self, l: int, r):
        """Mollified kernel M_l(r) = Phi_l(r)/r; M_l(0) = psi(0)/(c0 r_l)."""
        r = np.asarray(r, dtype=np.float64)
        rl = r_level(l)
        with np.errstate(divide="ignore", invalid="ignore"):
            out = self.psi.Phi(r / rl) / r
        return np.where(r == 0.0, self.psi.psi0 / (self.psi.c0 * rl), out)

    def M0_at_zero(self, l: int) -> float:
        """lim_{r->0} M_l(r): the self-interaction constant (Remark after Eq. 3.6,
        PAPER.md:524-541, for the PSWF split)."""
        return self.psi.psi0 / (self.psi.c0 * r_level(l))

    def D(self, l: int, r):
        """Difference kernel D_l = M_{l+1} - M_l (Eq. 3.66)."""
        return self.M(l + 1, r) - self.M(l, r)

    def R(self, l: int, r):
        """Residual kernel R_l(r) = (1 - Phi_l(r))/r (Eq. 3.66); zero for r >= r_l."""
        r = np.asarray(r, dtype=np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            out = (1.0 - self.psi.Phi(r / r_level(l))) / r
        return out

    # ---- Fourier space --------------------------------------------------
    def Dhat(self, l: int, k):
        """Eq. 3.68."""
        k = np.asarray(k, dtype=np.float64)
        c, p = self.c, self.psi
        rl, rl1 = r_level(l), r_level(l + 1)
        with np.errstate(divide="ignore", invalid="ignore"):
            v = 4.0 * np.pi / p.psi0 * (p(k * rl1 / c) - p(k * rl / c)) / k ** 2
        v0 = 2.0 * np.pi * p.c2 / p.c0 * (rl ** 2 - rl1 ** 2)
        return np.where(k == 0.0, v0, v)

    def What_root(self, k, RT: float):
        """Windowed M_1 at the root: psi(k r_1/c)/psi(0) * 8 pi sin^2(k RT/2)/k^2,
        value 2 pi RT^2 at k = 0 (reading R4)."""
        k = np.asarray(k, dtype=np.float64)
        p = self.psi
        G = p(k * r_level(1) / self.c) / p.psi0
        with np.errstate(divide="ignore", invalid="ignore"):
            T = 8.0 * np.pi * np.sin(k * RT / 2.0) ** 2 / k ** 2
        T = np.where(k == 0.0, 2.0 * np.pi * RT ** 2, T)
        return G * T


def trapezoid_weights_3d(fhat_radial, h: float, nf: int):
    """Weights w_m = (h/2pi)^3 fhat(h|m|) on m in [-nf, nf]^3 (Eq. 3.37 with the
    trapezoidal weight, reading R2).  Returned with axes (m1, m2, m3)."""
    m = np.arange(-nf, nf + 1, dtype=np.float64)
    kk = h * np.sqrt(m[:, None, None] ** 2 + m[None, :, None] ** 2 + m[None, None, :] ** 2)
    return (h / (2.0 * np.pi)) ** 3 * fhat_radial(kk)


def fourier_sum_3d(w, h: float, nf: int, x):
    """sum_m w_m e^{i h m . x} for points x (n,3): the spectral approximation of a
    radial kernel (Eq. 3.36).  Real part returned."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    m = np.arange(-nf, nf + 1, dtype=np.float64)
    e = [np.exp(1j * h * np.outer(x[:, d], m)) for d in range(3)]   # (n, N1)
    out = np.einsum("abc,na,nb,nc->n", w, e[0], e[1], e[2], optimize=True)
    return out.real
