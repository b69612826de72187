"""Pins for oracle/cheb.py (Sec. 2.1-2.2) and oracle/direct.py (Eq. 1.1)."""
import numpy as np
import pytest

from oracle import cheb, direct


@pytest.mark.parametrize("p", [9, 18, 28])
def test_nodes_are_roots_of_Tp(p):
    x = cheb.nodes(p)
    Tp = np.polynomial.chebyshev.chebval(x, [0] * p + [1])
    assert np.max(np.abs(Tp)) < 1e-13
    assert np.allclose(cheb.V(p) @ cheb.Vinv(p), np.eye(p), atol=1e-12)


@pytest.mark.parametrize("p", [9, 18])
def test_interpolation_exact_for_polynomials(p):
    rng = np.random.default_rng(0)
    coef = rng.standard_normal(p)                      # degree p-1
    f = lambda t: np.polynomial.chebyshev.chebval(t, coef)
    x = rng.uniform(-1, 1, 50)
    assert np.max(np.abs(cheb.interp_matrix(x, p) @ f(cheb.nodes(p)) - f(x))) < 1e-12


@pytest.mark.parametrize("p", [9, 18])
def test_proxy_charges_reproduce_polynomial_fields(p):
    """Def. 2.1: sum_j rho_j K(x_j) = sum_i rho~_i K(r_i) for any
    K of tensor degree < p, rho~ = U^T rho."""
    rng = np.random.default_rng(1)
    y = rng.uniform(-1, 1, (40, 3))
    rho = rng.uniform(-1, 1, 40)
    U = [cheb.interp_matrix(y[:, d], p) for d in range(3)]
    proxy = np.einsum("ja,jb,jc,j->abc", U[0], U[1], U[2], rho)
    c = [rng.standard_normal(p) for _ in range(3)]
    K1 = [lambda t, cc=cc: np.polynomial.chebyshev.chebval(t, cc) for cc in c]
    lhs = np.sum(rho * K1[0](y[:, 0]) * K1[1](y[:, 1]) * K1[2](y[:, 2]))
    r = cheb.nodes(p)
    rhs = np.einsum("abc,a,b,c->", proxy, K1[0](r), K1[1](r), K1[2](r))
    assert abs(lhs - rhs) < 1e-11 * np.sum(np.abs(rho))


@pytest.mark.parametrize("p", [9, 18])
def test_c2p_composes_with_anterpolation(p):
    """Lemma 2.2: child proxies then T_c2p == anterpolating the points on the parent."""
    rng = np.random.default_rng(2)
    sides = [-1, 1, -1]
    yc = rng.uniform(-1, 1, (30, 3))                   # child coordinates
    yp = yc / 2.0 + np.array(sides) * 0.5              # same points, parent coordinates
    rho = rng.uniform(-1, 1, 30)
    Uc = [cheb.interp_matrix(yc[:, d], p) for d in range(3)]
    Up = [cheb.interp_matrix(yp[:, d], p) for d in range(3)]
    child = np.einsum("ja,jb,jc,j->abc", *Uc, rho)
    direct_parent = np.einsum("ja,jb,jc,j->abc", *Up, rho)
    via = cheb.apply3([cheb.c2p_1d(p, s) for s in sides], child)
    assert np.max(np.abs(via - direct_parent)) < 1e-12


@pytest.mark.parametrize("p", [9, 18])
def test_p2c_exact(p):
    """Lemma 2.3: the child coefficients evaluate to the parent polynomial."""
    rng = np.random.default_rng(3)
    lam = rng.standard_normal((p, p, p))
    sides = [1, -1, 1]
    child = cheb.apply3([cheb.p2c_1d(p, s) for s in sides], lam)
    xc = rng.uniform(-1, 1, (20, 3))
    xp = xc / 2.0 + np.array(sides) * 0.5
    Ec = [cheb.vander(xc[:, d], p) for d in range(3)]
    Ep = [cheb.vander(xp[:, d], p) for d in range(3)]
    vc = np.einsum("ja,jb,jc,abc->j", *Ec, child)
    vp = np.einsum("ja,jb,jc,abc->j", *Ep, lam)
    assert np.max(np.abs(vc - vp)) < 1e-10 * np.max(np.abs(vp))


def shell_quadrature(R, nth=40):
    """Gauss-Legendre (cos theta) x trapezoid (phi) rule on the sphere of radius R;
    weights sum to the area 4 pi R^2 (exact for harmonics of degree < 2 nth)."""
    ct, wt = np.polynomial.legendre.leggauss(nth)
    nph = 2 * nth
    ph = 2 * np.pi * np.arange(nph) / nph
    st = np.sqrt(1 - ct ** 2)
    x = np.stack([np.outer(st, np.cos(ph)), np.outer(st, np.sin(ph)), np.outer(ct, np.ones(nph))], -1)
    w = np.outer(wt, np.full(nph, 2 * np.pi / nph)) * R ** 2
    return R * x.reshape(-1, 3), w.ravel()


def test_direct_uniform_shell_closed_form():
    """Uniformly charged spherical shell (total charge Q): potential Q/R inside,
    Q/|x| outside -- the closed form the direct sum must reproduce through a dense
    quadrature cloud (north-star oracle validation)."""
    R, Q = 0.3, 2.5
    y, w = shell_quadrature(R)
    q = Q * w / w.sum()
    rng = np.random.default_rng(4)
    inside = rng.uniform(-1, 1, (20, 3))
    inside *= (0.5 * R) / np.linalg.norm(inside, axis=1, keepdims=True) * rng.uniform(0, 1, (20, 1))
    outside = rng.standard_normal((20, 3))
    outside *= (2.0 * R + rng.uniform(0, 1, (20, 1))) / np.linalg.norm(outside, axis=1, keepdims=True)
    u_in = direct.laplace3d(y, q, inside)
    u_out = direct.laplace3d(y, q, outside)
    assert np.max(np.abs(u_in - Q / R)) < 1e-10 * Q / R
    assert np.max(np.abs(u_out - Q / np.linalg.norm(outside, axis=1))) < 1e-10 * Q / R


def test_direct_tiny_cases_and_self_exclusion():
    x = np.array([[0.0, 0.0, 0.0], [3.0, 4.0, 0.0], [0.0, 0.0, 0.0]])
    q = np.array([1.0, 2.0, 5.0])
    u = direct.laplace3d(x, q)
    # coincident points 0 and 2 do not interact; both see charge 2 at distance 5
    assert np.allclose(u, [2.0 / 5.0, (1.0 + 5.0) / 5.0, 2.0 / 5.0], rtol=0, atol=1e-15)
    assert np.all(direct.laplace3d(x, np.zeros(3)) == 0.0)
