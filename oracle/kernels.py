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


class YukawaSplit:
    """PSWF kernel split of the 3D Yukawa kernel K(r) = exp(-lam r)/r, carried out in
    Fourier space (Sec. 4.6, Eqs. 4.17-4.18):

        Khat(k)    = 4 pi/(k^2 + lam^2)        (the paper's 1/(k^2+lam^2) for the
                                                kernel normalised by 1/(4 pi), Eq. 4.16)
        Ghat_l(k)  = psi(sqrt(k^2+lam^2) r_l/c)/psi(0)
        Mhat_l     = Khat Ghat_l,   Dhat_l = Khat (Ghat_{l+1} - Ghat_l),
        Rhat_L     = Khat (1 - Ghat_L)                                (Eq. 4.18)

    In physical space M_l(r) is the radial inverse transform of Mhat_l (Eq. 3.12,
    PAPER.md:641): M_l(r) = 1/(2 pi^2 r) int_0^inf Mhat_l(k) k sin(kr) dk, taken over
    the support sqrt(k^2+lam^2) <= c/r_l of the truncated psi (reading R3) with
    Gauss-Legendre quadrature; R_L = K - M_L (no truncation: the oracle never assumes
    the compact support of R_L, it only computes it).
    Root (reading R4): the window of Sec. 4.7 with the truncated
    Yukawa kernel, That(k) = 4 pi int_0^{R_T} e^{-lam r} sin(kr)/k dr
      = 4 pi/(k^2+lam^2) [1 - e^{-lam R_T}(cos k R_T + (lam/k) sin k R_T)].
    lam is the Yukawa parameter in the units of the coordinates the split is used in
    (oracle/dmk.py passes lam * side for the unit root cube)."""

    NQ = 400

    def __init__(self, c: float, lam: float):
        if not lam > 0:
            raise ValueError("YukawaSplit needs lam > 0 (lam = 0 is LaplaceSplit)")
        self.psi = Pswf(c)
        self.c = self.psi.c
        self.lam = float(lam)
        self._gl = np.polynomial.legendre.leggauss(self.NQ)

    def K(self, r):
        r = np.asarray(r, dtype=np.float64)
        with np.errstate(divide="ignore"):
            return np.exp(-self.lam * r) / r

    def Khat(self, k):
        k = np.asarray(k, dtype=np.float64)
        return 4.0 * np.pi / (k ** 2 + self.lam ** 2)

    def Ghat(self, l: int, k):
        k = np.asarray(k, dtype=np.float64)
        return self.psi(np.sqrt(k ** 2 + self.lam ** 2) * r_level(l) / self.c) / self.psi.psi0

    def Dhat(self, l: int, k):
        """Eq. 4.18, second line (times 4 pi)."""
        return self.Khat(k) * (self.Ghat(l + 1, k) - self.Ghat(l, k))

    def What_root(self, k, RT: float):
        k = np.asarray(k, dtype=np.float64)
        lam = self.lam
        with np.errstate(divide="ignore", invalid="ignore"):
            T = 4.0 * np.pi / (k ** 2 + lam ** 2) * (
                1.0 - np.exp(-lam * RT) * (np.cos(k * RT) + lam / k * np.sin(k * RT)))
        T0 = 4.0 * np.pi / lam ** 2 * (1.0 - np.exp(-lam * RT) * (1.0 + lam * RT))
        return self.Ghat(1, k) * np.where(k == 0.0, T0, T)

    def _kgrid(self, l: int):
        kmax2 = (self.c / r_level(l)) ** 2 - self.lam ** 2
        if kmax2 <= 0:
            return None, None
        x, w = self._gl
        kmax = np.sqrt(kmax2)
        return 0.5 * kmax * (x + 1.0), 0.5 * kmax * w

    def M(self, l: int, r):
        """Mollified kernel M_l(r) by the radial inverse Fourier transform."""
        r = np.asarray(r, dtype=np.float64)
        k, w = self._kgrid(l)
        if k is None:
            return np.zeros_like(r)
        f = self.Khat(k) * self.Ghat(l, k) * w
        flat = r.reshape(-1)
        out = np.empty_like(flat)
        for a in range(0, flat.size, 4096):
            rr = flat[a:a + 4096]
            kr = np.outer(rr, k)
            with np.errstate(divide="ignore", invalid="ignore"):
                s = np.where(kr > 0, np.sin(kr) / np.where(kr > 0, kr, 1.0), 1.0)
            out[a:a + 4096] = (s * (f * k ** 2)[None, :]).sum(axis=1) / (2.0 * np.pi ** 2)
        return out.reshape(r.shape)

    def M0_at_zero(self, l: int) -> float:
        return float(self.M(l, np.array([0.0]))[0])

    def D(self, l: int, r):
        return self.M(l + 1, r) - self.M(l, r)

    def R(self, l: int, r):
        """Residual kernel R_l = K - M_l (r > 0)."""
        r = np.asarray(r, dtype=np.float64)
        return self.K(r) - self.M(l, r)


def trapezoid_weights(fhat_radial, h: float, nf: int, d: int):
    """Weights (h/2pi)^d fhat(h|m|) on m in [-nf, nf]^d (Eq. 3.37, reading R2)."""
    if d == 3:
        return trapezoid_weights_3d(fhat_radial, h, nf)
    m = np.arange(-nf, nf + 1, dtype=np.float64)
    kk = h * np.sqrt(m[:, None] ** 2 + m[None, :] ** 2)
    return (h / (2.0 * np.pi)) ** 2 * fhat_radial(kk)


def fourier_sum_2d(w, h: float, nf: int, x):
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    m = np.arange(-nf, nf + 1, dtype=np.float64)
    e = [np.exp(1j * h * np.outer(x[:, d], m)) for d in range(2)]
    return np.einsum("ab,na,nb->n", w, e[0], e[1], optimize=True).real


class LogSplit2D:
    """PSWF kernel split of the 2D kernel K(r) = -log r in Fourier space (Sec. 4.6,
    PAPER.md:2441-2447: Eq. 4.18 with lam = 0 "provides an efficient kernel splitting
    for ... log(r)"):

        Khat(k) = 2 pi/k^2 (-log r = 2 pi G_L, Ghat_L = 1/k^2, Eq. 4.16 in 2D)
        Ghat_l(k) = psi(k r_l/c)/psi(0),  Dhat_l = Khat (Ghat_{l+1} - Ghat_l)
        Dhat_l(0) = pi (c2/c0) (r_l^2 - r_{l+1}^2)

    (the k -> 0 limit, with psi''(0)/psi(0) = -c^2 c2/c0 as in Eq. 3.68).  In physical
    space (2D radial inverse transform f(r) = 1/(2 pi) int fhat(k) J_0(kr) k dk):
        M_l(r) = M_l(0) + int_0^{c/r_l} Ghat_l(k) (J_0(kr) - 1)/k dk,
        M_l(0) = -log r_l + log(c/2) + gamma + int_0^1 (psi(x)/psi(0) - 1)/x dx,
    the constant being the one for which M_l(r) + log r -> 0 as r -> inf (the
    distributional transform of -log r; uses int_0^X (1 - J_0(u))/u du = log(X/2) +
    gamma + o(1)).  R_L = K - M_L.  Root window (reading R4, Sec. 4.7): the transform of
    -log r truncated at R_T,
        That(k) = 2 pi (1 - J_0(k R_T))/k^2 - 2 pi R_T log(R_T) J_1(k R_T)/k,
        That(0) = pi R_T^2/2 - pi R_T^2 log R_T."""

    NQ = 400

    def __init__(self, c: float):
        from scipy.special import j0, j1
        self._j0, self._j1 = j0, j1
        self.psi = Pswf(c)
        self.c = self.psi.c
        x, w = np.polynomial.legendre.leggauss(self.NQ)
        self._gx, self._gw = 0.5 * (x + 1.0), 0.5 * w          # on [0, 1]
        g = self.psi(self._gx) / self.psi.psi0
        self.kappa = np.log(self.c / 2.0) + np.euler_gamma + np.sum(self._gw * (g - 1.0) / self._gx)

    def K(self, r):
        r = np.asarray(r, dtype=np.float64)
        with np.errstate(divide="ignore"):
            return -np.log(r)

    def Ghat(self, l: int, k):
        return self.psi(np.asarray(k, dtype=np.float64) * r_level(l) / self.c) / self.psi.psi0

    def Dhat(self, l: int, k):
        k = np.asarray(k, dtype=np.float64)
        p = self.psi
        rl, rl1 = r_level(l), r_level(l + 1)
        with np.errstate(divide="ignore", invalid="ignore"):
            v = 2.0 * np.pi * (self.Ghat(l + 1, k) - self.Ghat(l, k)) / k ** 2
        v0 = np.pi * p.c2 / p.c0 * (rl ** 2 - rl1 ** 2)
        return np.where(k == 0.0, v0, v)

    def What_root(self, k, RT: float):
        k = np.asarray(k, dtype=np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            T = (2.0 * np.pi * (1.0 - self._j0(k * RT)) / k ** 2
                 - 2.0 * np.pi * RT * np.log(RT) * self._j1(k * RT) / k)
        T0 = np.pi * RT ** 2 / 2.0 - np.pi * RT ** 2 * np.log(RT)
        return self.Ghat(1, k) * np.where(k == 0.0, T0, T)

    def M0_at_zero(self, l: int) -> float:
        return -np.log(r_level(l)) + self.kappa

    def M(self, l: int, r):
        r = np.asarray(r, dtype=np.float64)
        kmax = self.c / r_level(l)
        k, w = kmax * self._gx, kmax * self._gw
        f = w * self.Ghat(l, k) / k
        flat = r.reshape(-1)
        out = np.empty_like(flat)
        for a in range(0, flat.size, 4096):
            kr = np.outer(flat[a:a + 4096], k)
            out[a:a + 4096] = ((self._j0(kr) - 1.0) * f[None, :]).sum(axis=1)
        return out.reshape(r.shape) + self.M0_at_zero(l)

    def D(self, l: int, r):
        return self.M(l + 1, r) - self.M(l, r)

    def R(self, l: int, r):
        r = np.asarray(r, dtype=np.float64)
        return self.K(r) - self.M(l, r)
