"""Prolate spheroidal wave function of order zero, psi_0^c  (oracle; test infrastructure).

PAPER.md:3144-3175 (App. A.5): psi_0^c is the eigenfunction of
    F_c[phi](x) = int_{-1}^{1} phi(t) e^{i c x t} dt        (Eq. A.15)
with the largest |eigenvalue| lambda_0; it is real, even, has no roots in (-1,1)
and is L2-normalised on [-1,1].  The paper cites [osipov2013] without fixing a
method.  We use the classical fact that psi_0^c is also the lowest eigenfunction
of the prolate differential operator
    L psi = -((1-x^2) psi')' + c^2 x^2 psi,
which is symmetric tridiagonal in the normalised Legendre basis
Pbar_n = sqrt(n+1/2) P_n (even n only for psi_0).  This construction is NOT
pinned by re-using it: tests/test_oracle_pswf.py checks the integral-operator
eigen-equation Eq. A.15 by direct Gauss-Legendre quadrature and the Fig. 6
caption value psi(1)/psi(0) = 1e-6 at c = 16.893999099731445.

Truncation ("if we truncate psi at +-c"): the function is
taken to be zero for |x| > 1.  This is reading R3 in DESIGN.md.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as npleg


class Pswf:
    """psi_0^c on [-1,1] as a Legendre series.  Attributes:

    c        band-limit parameter
    coef     coefficients in the *plain* Legendre basis P_n (numpy legendre order)
    lambda0  eigenvalue of F_c (real, positive for n = 0)
    psi0     psi(0)
    c0       int_0^1 psi(x) dx
    c2       int_0^1 x^2 psi(x) dx
    """

    def __init__(self, c: float, nmax: int | None = None):
        self.c = float(c)
        if nmax is None:
            nmax = 2 * int(np.ceil(self.c)) + 60
        ns = np.arange(0, nmax + 1, 2, dtype=np.float64)   # even degrees only
        m = len(ns)
        A = np.zeros((m, m))
        for k, n in enumerate(ns):
            b = (2 * n * (n + 1) - 1) / ((2 * n + 3) * (2 * n - 1))   # <Pbar_n, x^2 Pbar_n>
            A[k, k] = n * (n + 1) + self.c ** 2 * b
            if k + 1 < m:
                a = (n + 1) * (n + 2) / ((2 * n + 3) * np.sqrt((2 * n + 1) * (2 * n + 5)))
                A[k, k + 1] = A[k + 1, k] = self.c ** 2 * a          # <Pbar_{n+2}, x^2 Pbar_n>
        w, v = np.linalg.eigh(A)
        beta = v[:, 0]                       # lowest eigenvalue -> psi_0; unit 2-norm = L2 norm 1
        coef = np.zeros(nmax + 1)
        coef[0::2] = beta * np.sqrt(ns + 0.5)          # Pbar_n -> P_n
        if npleg.legval(0.0, coef) < 0:
            coef = -coef
        self.coef = coef
        self.chi0 = w[0]
        self.psi0 = float(npleg.legval(0.0, coef))
        # antiderivative with value 0 at x = 0 (psi even -> antiderivative odd)
        self._int = npleg.legint(coef, lbnd=0.0)
        self.c0 = float(npleg.legval(1.0, self._int))
        # int_{-1}^{1} psi = 2 c0 = lambda0 psi(0)   (F_c at x=0, Eq. A.15)
        self.lambda0 = 2.0 * self.c0 / self.psi0
        x2 = npleg.legmulx(npleg.legmulx(coef))
        self.c2 = float(npleg.legval(1.0, npleg.legint(x2, lbnd=0.0)))

    def __call__(self, x):
        """psi_0^c(x), truncated to zero for |x| > 1 (reading R3)."""
        x = np.asarray(x, dtype=np.float64)
        out = npleg.legval(np.clip(x, -1.0, 1.0), self.coef)
        return np.where(np.abs(x) <= 1.0, out, 0.0)

    def integral(self, x):
        """int_0^x psi(t) dt for x in [-1, 1]; constant beyond (truncation)."""
        x = np.clip(np.asarray(x, dtype=np.float64), -1.0, 1.0)
        return npleg.legval(x, self._int)

    def Phi(self, t):
        """Phi(t) = (1/c0) int_0^t psi, t >= 0; equal to 1 for t >= 1.
        PAPER.md:1944-1946 (definition of Phi^c_l with t = r / r_l)."""
        t = np.asarray(t, dtype=np.float64)
        return np.where(t >= 1.0, 1.0, self.integral(np.minimum(t, 1.0)) / self.c0)
