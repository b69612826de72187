"""Pins for oracle/kernels.py and oracle/params.py (PSWF split of 1/r, Sec. 3.6)."""
import json
import os

import numpy as np
import pytest

from oracle import params
from oracle.kernels import LaplaceSplit, fourier_sum_3d, r_level, trapezoid_weights_3d

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EPS = [1e-3, 1e-6, 1e-9]


def radial_ft_3d(f, rmax, k, breaks=()):
    """fhat(k) = 4 pi int_0^rmax sin(kr)/(kr) f(r) r^2 dr  (Eq. A.4),
    composite Gauss-Legendre on [0, rmax] split at `breaks`."""
    pts = [0.0] + sorted(breaks) + [rmax]
    x, w = np.polynomial.legendre.leggauss(200)
    tot = np.zeros_like(k, dtype=np.float64)
    for a, b in zip(pts, pts[1:]):
        r = 0.5 * (b - a) * (x + 1) + a
        ww = 0.5 * (b - a) * w
        kr = np.outer(k, r)
        sinc = np.where(kr == 0, 1.0, np.sin(kr) / np.where(kr == 0, 1, kr))
        tot += (sinc * (f(r) * r ** 2 * ww)[None, :]).sum(axis=1)
    return 4 * np.pi * tot


@pytest.mark.parametrize("eps", EPS)
@pytest.mark.parametrize("l", [0, 1, 3])
def test_difference_kernel_ft_matches_radial_transform(eps, l):
    """Eq. 3.68 vs the radial Fourier transform of D_l computed in physical space."""
    S = LaplaceSplit(params.for_eps(eps).c)
    k = np.linspace(0.0, 2.2 * S.c / r_level(l), 41)
    num = radial_ft_3d(lambda r: S.D(l, r), r_level(l), k, breaks=[r_level(l + 1)])
    ana = S.Dhat(l, k)
    scale = np.max(np.abs(ana))
    assert np.max(np.abs(num - ana)) <= 20 * eps * scale


@pytest.mark.parametrize("eps", EPS)
def test_dhat_zero_branch_is_limit(eps):
    """Second line of Eq. 3.68 (D_l(0) via c2/c0) equals the k->0 limit of the first."""
    S = LaplaceSplit(params.for_eps(eps).c)
    for l in (0, 2):
        k1 = 0.02 / r_level(l)
        d1, d2 = S.Dhat(l, np.array([k1, 2 * k1]))
        limit = (4 * d1 - d2) / 3.0          # Richardson: Dhat(k) = a + b k^2 + O(k^4)
        assert abs(limit - S.Dhat(l, np.array([0.0]))[0]) < 1e-7 * abs(limit)


@pytest.mark.parametrize("eps", EPS)
def test_root_window_equals_mollified_kernel(eps):
    """Windowed kernel What (truncated 1/r, Sec. 4.7) inverted radially equals M_1
    on r <= sqrt(3) (Eq. 4.21 / Lemma 3.2 analogue)."""
    prm = params.for_eps(eps)
    S = LaplaceSplit(prm.c)
    r = np.linspace(0.05, np.sqrt(3.0), 23)
    kmax = 2 * S.c / r_level(0) * 1.05
    x, w = np.polynomial.legendre.leggauss(400)
    pts = np.linspace(0, kmax, 41)
    tot = np.zeros_like(r)
    for a, b in zip(pts, pts[1:]):
        k = 0.5 * (b - a) * (x + 1) + a
        ww = 0.5 * (b - a) * w
        F = S.What_root(k, prm.RT)
        tot += (np.sin(np.outer(r, k)) / np.outer(r, k) * (F * k ** 2 * ww)[None, :]).sum(axis=1)
    W = tot / (2 * np.pi ** 2)            # Eq. 3.12 inverse radial transform
    assert np.max(np.abs(W - S.M(1, r))) <= 10 * eps * S.M(1, 0.0)


@pytest.mark.parametrize("row", json.load(open(os.path.join(GOLD, "table1.json")))["rows"][:3])
def test_table1_fourier_and_order_reach_eps(row):
    """Table 1's N_1 = 2 n_f + 1 with spacing 2 pi/(3 r_l) resolves D_l on the
    colleague range |x|_inf < 2 r_l to eps (SPEC acceptance 2, reading R2)."""
    eps, c, N1 = row[0], row[1], row[2]
    prm = params.for_eps(eps)
    assert prm.c == c and 2 * prm.nf + 1 == N1 and prm.p == row[3]
    S = LaplaceSplit(c)
    rng = np.random.default_rng(3)
    for l in (1, 4):
        rl = r_level(l)
        x = rng.uniform(-2 * rl, 2 * rl, (300, 3))
        h = prm.h(l)
        w = trapezoid_weights_3d(lambda k: S.Dhat(l, k), h, prm.nf)
        err = np.max(np.abs(fourier_sum_3d(w, h, prm.nf, x) - S.D(l, np.linalg.norm(x, axis=1))))
        assert err <= 2 * eps * S.D(l, 0.0)


@pytest.mark.parametrize("eps", EPS)
def test_telescoping_identity_with_fourier_pieces(eps):
    """1/r = W_0 + sum_{l<L} D_l + R_L with the window and the
    difference kernels evaluated through their trapezoidal Fourier sums and R_L in
    physical space, at sampled x in the range each level handles."""
    prm = params.for_eps(eps)
    S = LaplaceSplit(prm.c)
    rng = np.random.default_rng(5)
    for L in (1, 2, 4):
        lim = 1.0 if L == 1 else 2 * r_level(L - 1)
        x = rng.uniform(-lim, lim, (200, 3))
        r = np.linalg.norm(x, axis=1)
        h0 = prm.h(0)
        tot = fourier_sum_3d(trapezoid_weights_3d(lambda k: S.What_root(k, prm.RT), h0, prm.nf0), h0, prm.nf0, x)
        for l in range(1, L):
            h = prm.h(l)
            tot += fourier_sum_3d(trapezoid_weights_3d(lambda k, l=l: S.Dhat(l, k), h, prm.nf), h, prm.nf, x)
        tot += S.R(L, r)
        assert np.max(np.abs(tot - 1.0 / r)) <= 3 * eps * S.M(L, 0.0)


@pytest.mark.parametrize("eps", EPS)
def test_compact_support_and_self_constant(eps):
    S = LaplaceSplit(params.for_eps(eps).c)
    for l in (1, 3):
        rl = r_level(l)
        r = np.linspace(rl, 2 * rl, 50)
        assert np.all(S.R(l, r) == 0.0) and np.all(S.D(l, r) == 0.0)
        # residual decays to ~eps * scale at r -> r_l (Phi(1) = 1)
        assert abs(S.R(l, rl * (1 - 1e-9))) < 1e-6 / rl
        # M_l(0) = psi(0)/(c0 r_l) is the r -> 0 limit (self-interaction constant)
        assert abs(S.M(l, 1e-9 * rl) - S.M0_at_zero(l)) < 1e-9 * S.M0_at_zero(l)


def test_precision_snaps_to_next_tighter_row():
    """Reading R1: a requested eps between Table 1 rows uses the next tighter row."""
    assert params.for_eps(2e-6).eps == 1e-6 and params.for_eps(1e-3).eps == 1e-3
    assert params.for_eps(0.5).eps == 1e-3 and params.for_eps(5e-8).eps == 1e-9
    with pytest.raises(ValueError):
        params.for_eps(1e-13)
