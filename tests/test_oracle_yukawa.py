"""Pins for the Yukawa oracle (oracle/kernels.py YukawaSplit, oracle/direct.py
yukawa3d, oracle/dmk.py dmk_yukawa3d): Sec. 4.6, Eqs. 4.17-4.18
and the window construction of Sec. 4.7."""
import numpy as np
import pytest

import dmk_inputs
from oracle import direct, params
from oracle.dmk import dmk_yukawa3d
from oracle.kernels import LaplaceSplit, YukawaSplit, fourier_sum_3d, r_level, trapezoid_weights_3d

EPS = [1e-3, 1e-6, 1e-9]
LAM = 10.0


def fibonacci_sphere(n, radius, centre):
    i = np.arange(n) + 0.5
    z = 1.0 - 2.0 * i / n
    phi = np.pi * (1.0 + 5 ** 0.5) * i
    rr = np.sqrt(1.0 - z * z)
    return centre + radius * np.stack([rr * np.cos(phi), rr * np.sin(phi), z], axis=1)


def test_direct_sum_uniform_shell_closed_form():
    """A uniformly charged spherical shell (radius a, total charge Q) has the Yukawa
    potential Q e^{-lam d} sinh(lam a)/(lam a d) outside and Q e^{-lam a} sinh(lam d)/
    (lam a d) inside (distance d from the centre): closed forms of the sphere average of
    e^{-lam|x-y|}/|x-y|.  The direct sum over a dense equal-weight Fibonacci cloud
    reproduces them to quadrature accuracy."""
    a, Q, c = 0.3, 2.0, np.array([0.5, 0.5, 0.5])
    y = fibonacci_sphere(60000, a, c)
    q = np.full(len(y), Q / len(y))
    d = np.array([0.5, 0.7, 1.1, 0.05, 0.12, 0.2])
    dirs = np.random.default_rng(0).standard_normal((len(d), 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    x = c + d[:, None] * dirs
    got = direct.yukawa3d(y, q, LAM, targets=x)
    out = d > a
    ref = np.where(out, Q * np.exp(-LAM * d) * np.sinh(LAM * a) / (LAM * a * d),
                   Q * np.exp(-LAM * a) * np.sinh(LAM * d) / (LAM * a * d))
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-4


def test_direct_sum_lambda_zero_is_laplace_and_tiny_brute_force():
    x, q = dmk_inputs.uniform(50, seed=1)
    assert np.allclose(direct.yukawa3d(x, q, 0.0), direct.laplace3d(x, q), rtol=1e-14)
    i, j = 3, 17
    r = np.linalg.norm(x[i] - x[j])
    two = direct.yukawa3d(x[[i, j]], q[[i, j]], 2.5)
    assert np.isclose(two[0], q[j] * np.exp(-2.5 * r) / r, rtol=1e-14)


def test_truncated_kernel_transform_closed_form():
    """That(k) of the root window equals 4 pi/k int_0^R e^{-lam r} sin(kr) dr."""
    Y = YukawaSplit(params.for_eps(1e-6).c, 7.0)
    R = 1.0 + np.sqrt(3.0)
    k = np.array([1e-3, 0.5, 3.0, 11.0, 20.0])   # inside the support of Ghat_1
    x, w = np.polynomial.legendre.leggauss(400)
    pts = np.linspace(0, R, 21)
    num = np.zeros_like(k)
    for a, b in zip(pts, pts[1:]):
        r = 0.5 * (b - a) * (x + 1) + a
        num += (np.exp(-7.0 * r)[None, :] * np.sin(np.outer(k, r)) * (0.5 * (b - a) * w)[None, :]).sum(1)
    num *= 4 * np.pi / k
    ana = Y.What_root(k, R) / Y.Ghat(1, k)
    assert np.max(np.abs(num - ana) / np.abs(ana)) < 1e-10
    # k -> 0 branch is the limit
    assert np.isclose(Y.What_root(np.array([0.0]), R)[0] / Y.Ghat(1, np.array([0.0]))[0],
                      ana[0], rtol=1e-6)


@pytest.mark.parametrize("eps", EPS)
def test_lambda_to_zero_reduces_to_laplace_split(eps):
    """Eq. 4.18 with lam -> 0 is Eq. 3.68 (the paper's remark): the
    radially inverted mollifier equals the physical-space Laplace M_l = Phi_l/r."""
    c = params.for_eps(eps).c
    Y, L = YukawaSplit(c, 1e-9), LaplaceSplit(c)
    for l in (0, 2):
        r = np.linspace(0.0, 1.5 * r_level(l), 31)
        assert np.max(np.abs(Y.M(l, r) - L.M(l, r))) <= 2 * eps * L.M0_at_zero(l)
        k = np.linspace(0.05, 1.5, 17) * c / r_level(l)   # k = 0 is singular as lam -> 0
        assert np.max(np.abs(Y.Dhat(l, k) - L.Dhat(l, k))) <= 1e-6 * np.max(np.abs(L.Dhat(l, k)))


@pytest.mark.parametrize("eps", EPS)
def test_residual_compactly_supported(eps):
    """R_L = K - M_L is negligible beyond r_L: M_L reproduces the
    Yukawa kernel there, which pins the mollifier to K itself."""
    Y = YukawaSplit(params.for_eps(eps).c, LAM)
    for l in (2, 3, 5):
        rl = r_level(l)
        r = np.linspace(rl, 3 * rl, 25)
        assert np.max(np.abs(Y.R(l, r))) <= 2 * eps * Y.M0_at_zero(l)


@pytest.mark.parametrize("eps", EPS)
def test_root_window_equals_mollified_kernel(eps):
    """The windowed kernel (truncated Yukawa, Sec. 4.7) equals M_1 on r <= sqrt 3."""
    prm = params.for_eps(eps)
    Y = YukawaSplit(prm.c, LAM)
    r = np.linspace(0.05, np.sqrt(3.0), 19)
    kmax = 2 * Y.c * 1.05
    x, w = np.polynomial.legendre.leggauss(400)
    pts = np.linspace(0, kmax, 41)
    tot = np.zeros_like(r)
    for a, b in zip(pts, pts[1:]):
        k = 0.5 * (b - a) * (x + 1) + a
        ww = 0.5 * (b - a) * w
        tot += (np.sin(np.outer(r, k)) / np.outer(r, k) * (Y.What_root(k, prm.RT) * k ** 2 * ww)[None, :]).sum(1)
    W = tot / (2 * np.pi ** 2)
    assert np.max(np.abs(W - Y.M(1, r))) <= 10 * eps * Y.M0_at_zero(1)


@pytest.mark.parametrize("eps", EPS)
def test_telescoping_identity_with_fourier_pieces(eps):
    """K = W_0 + sum_{l<L} D_l + R_L with W_0, D_l through their trapezoidal Fourier
    sums (the device's representation) and R_L = K - M_L in physical space."""
    prm = params.for_eps(eps)
    Y = YukawaSplit(prm.c, LAM)
    rng = np.random.default_rng(5)
    for L in (1, 3):
        lim = 1.0 if L == 1 else 2 * r_level(L - 1)
        x = rng.uniform(-lim, lim, (120, 3))
        r = np.linalg.norm(x, axis=1)
        h0 = prm.h(0)
        tot = fourier_sum_3d(trapezoid_weights_3d(lambda k: Y.What_root(k, prm.RT), h0, prm.nf0), h0, prm.nf0, x)
        for l in range(1, L):
            h = prm.h(l)
            tot += fourier_sum_3d(trapezoid_weights_3d(lambda k, l=l: Y.Dhat(l, k), h, prm.nf), h, prm.nf, x)
        tot += Y.R(L, r)
        assert np.max(np.abs(tot - Y.K(r))) <= 3 * eps * Y.M0_at_zero(L)


@pytest.mark.parametrize("eps", [1e-3, 1e-6])
def test_dmk_yukawa_matches_direct_sum(eps):
    x, q = dmk_inputs.clusters(2000, seed=3)
    u = dmk_yukawa3d(x, q, eps, 30, LAM)
    assert direct.rel_l2(u, direct.yukawa3d(x, q, LAM)) <= 2 * eps
