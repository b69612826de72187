"""Pins for the 2D log oracle (oracle/kernels.py LogSplit2D, oracle/direct.py log2d,
oracle/tree.py with d = 2, oracle/dmk.py dmk_log2d): the Fourier-space PSWF split of
Sec. 4.6 at lam = 0 in 2D, window of Sec. 4.7."""
import itertools

import numpy as np
import pytest
from scipy.special import j0

import dmk_inputs
from oracle import direct, params
from oracle.dmk import dmk_log2d
from oracle.kernels import LogSplit2D, fourier_sum_2d, r_level, trapezoid_weights
from oracle.tree import NBITS, Tree, morton

EPS = [1e-3, 1e-6, 1e-9]


def noisy_circle(n, seed):
    """BASELINE config 3's distribution: radius 0.4 + N(0, 1e-3) about (0.5, 0.5),
    charges U[-1,1] with zero mean."""
    return dmk_inputs.circle2d(n, seed=seed)


def test_direct_sum_ring_closed_form():
    """A uniformly charged ring (radius a, charge Q) has the 2D potential
    -Q log max(d, a) at distance d from its centre (mean-value property of log|x|);
    equally spaced points give the trapezoidal rule, spectrally accurate off the ring."""
    a, Q, c = 0.3, 1.7, np.array([0.4, 0.6])
    n = 4000
    th = 2 * np.pi * np.arange(n) / n
    y = c + a * np.stack([np.cos(th), np.sin(th)], 1)
    q = np.full(n, Q / n)
    d = np.array([0.05, 0.2, 0.35, 0.9, 2.5])
    x = c + d[:, None] * np.array([[np.cos(0.3), np.sin(0.3)]])
    got = direct.log2d(y, q, targets=x)
    assert np.allclose(got, -Q * np.log(np.maximum(d, a)), rtol=0, atol=1e-12)


def test_morton_2d_and_quadtree_structure():
    q = np.random.default_rng(0).integers(0, 2 ** NBITS, (100, 2))
    brute = [sum((((int(r[k]) >> b) & 1) << (2 * b + (1 - k))) for b in range(NBITS) for k in range(2)) for r in q]
    assert np.array_equal(morton(q), np.array(brute, dtype=np.int64))
    x = np.array([[a, b] for a in (0.25, 0.75) for b in (0.25, 0.75)])
    T = Tree(x, 1)
    assert T.d == 2 and T.nbox == 5 and T.nlevels == 2 and np.sum(T.box_leaf) == 4


@pytest.mark.parametrize("kind", ["uniform", "circle"])
def test_quadtree_balance_colleagues_and_lists(kind):
    x = (dmk_inputs.uniform(2000, seed=2, dim=2)[0] if kind == "uniform" else noisy_circle(2000, 2)[0])
    T = Tree(x, 15)
    leaves = np.nonzero(T.box_leaf)[0]
    assert np.all(T.box_npts[leaves] <= 15) or np.max(T.box_level) == 20
    # colleagues: same level, |coord diff|_inf <= 1, slot order of itertools.product
    for i in range(0, T.nbox, 7):
        for k, off in enumerate(itertools.product((-1, 0, 1), repeat=2)):
            j = T.box_colleagues[i, k]
            if j >= 0:
                assert T.box_level[j] == T.box_level[i]
                assert np.array_equal(T.box_coords[j] - T.box_coords[i], off)
    # 2:1 balance: touching leaves differ by at most one level
    s = 2.0 ** -T.box_level[leaves]
    lo = T.box_coords[leaves] * s[:, None]
    for a in range(len(leaves)):
        touch = np.all((lo[a] <= lo + s[:, None]) & (lo <= lo[a] + s[a]), axis=1)
        assert np.all(np.abs(T.box_level[leaves][touch] - T.box_level[leaves[a]]) <= 1)
    # direct lists complete: every pair of non-empty leaves closer than the larger
    # residual range must be listed (brute force over leaf pairs)
    ne = [i for i in leaves if T.box_npts[i] > 0]
    for i in ne[::5]:
        for j in ne:
            si, sj = 2.0 ** -T.box_level[i], 2.0 ** -T.box_level[j]
            li, lj = T.box_coords[i] * si, T.box_coords[j] * sj
            gap = np.linalg.norm(np.maximum(0, np.maximum(li - (lj + sj), lj - (li + si))))
            if gap < min(sj, si) * 0.999 and T.box_level[j] <= T.box_level[i]:
                assert j in T.dlist[i]


@pytest.mark.parametrize("eps", EPS)
def test_dhat_zero_branch_and_scale_invariance(eps):
    S = LogSplit2D(params.for_eps(eps, 2).c)
    for l in (0, 2):
        k1 = 0.02 / r_level(l)
        d1, d2 = S.Dhat(l, np.array([k1, 2 * k1]))
        assert abs((4 * d1 - d2) / 3.0 - S.Dhat(l, np.array([0.0]))[0]) < 1e-7 * abs(d1)
    r = np.linspace(0, 1.3, 11)
    assert np.allclose(S.M(3, r * r_level(3)) + np.log(r_level(3)), S.M(0, r), rtol=0, atol=1e-12)


@pytest.mark.parametrize("eps", EPS)
def test_residual_compactly_supported_pins_constant(eps):
    """R_L = -log r - M_L vanishes beyond r_L to eps.  A wrong
    M_L(0) constant (the distributional part of the log transform) fails this."""
    S = LogSplit2D(params.for_eps(eps, 2).c)
    for l in (0, 2, 5):
        r = np.linspace(1.0, 4.0, 31) * r_level(l)
        assert np.max(np.abs(S.R(l, r))) <= 2 * eps


@pytest.mark.parametrize("eps", EPS)
def test_difference_kernel_hankel_transform(eps):
    """Dhat_l(k) = 2 pi int_0^{r_l} D_l(r) J_0(kr) r dr (2D radial transform of the
    physical-space difference kernel)."""
    S = LogSplit2D(params.for_eps(eps, 2).c)
    l = 1
    rl = r_level(l)
    x, w = np.polynomial.legendre.leggauss(300)
    pts = np.linspace(0, 1.2 * rl, 13)
    rr, ww = [], []
    for a, b in zip(pts, pts[1:]):
        rr.append(0.5 * (b - a) * (x + 1) + a)
        ww.append(0.5 * (b - a) * w)
    rr, ww = np.concatenate(rr), np.concatenate(ww)
    Dr = S.D(l, rr)
    k = np.linspace(0.0, 1.5 * S.c / rl, 23)
    num = 2 * np.pi * (j0(np.outer(k, rr)) * (Dr * rr * ww)[None, :]).sum(1)
    ana = S.Dhat(l, k)
    assert np.max(np.abs(num - ana)) <= 50 * eps * np.max(np.abs(ana))


@pytest.mark.parametrize("eps", EPS)
def test_root_window_equals_mollified_kernel(eps):
    """The windowed kernel (-log r truncated at R_T = (1 + sqrt 2) r_0) inverted radially
    equals M_1 on r <= sqrt 2."""
    prm = params.for_eps(eps, 2)
    S = LogSplit2D(prm.c)
    r = np.linspace(0.05, np.sqrt(2.0), 17)
    kmax = 2 * S.c * 1.02
    x, w = np.polynomial.legendre.leggauss(400)
    pts = np.linspace(0, kmax, 61)
    tot = np.zeros_like(r)
    for a, b in zip(pts, pts[1:]):
        k = 0.5 * (b - a) * (x + 1) + a
        tot += (j0(np.outer(r, k)) * (S.What_root(k, prm.RT) * k * 0.5 * (b - a) * w)[None, :]).sum(1)
    W = tot / (2 * np.pi)
    assert np.max(np.abs(W - S.M(1, r))) <= 20 * eps


@pytest.mark.parametrize("eps", EPS)
def test_telescoping_identity_with_fourier_pieces(eps):
    prm = params.for_eps(eps, 2)
    S = LogSplit2D(prm.c)
    rng = np.random.default_rng(5)
    for L in (1, 3):
        lim = 1.0 if L == 1 else 2 * r_level(L - 1)
        x = rng.uniform(-lim, lim, (150, 2))
        r = np.linalg.norm(x, axis=1)
        h0 = prm.h(0)
        tot = fourier_sum_2d(trapezoid_weights(lambda k: S.What_root(k, prm.RT), h0, prm.nf0, 2), h0, prm.nf0, x)
        for l in range(1, L):
            h = prm.h(l)
            tot += fourier_sum_2d(trapezoid_weights(lambda k, l=l: S.Dhat(l, k), h, prm.nf, 2), h, prm.nf, x)
        tot += S.R(L, r)
        assert np.max(np.abs(tot - S.K(r))) <= 4 * eps


@pytest.mark.parametrize("eps", EPS)
def test_dmk_log2d_matches_direct(eps):
    x, q = noisy_circle(3000, 3)
    assert direct.rel_l2(dmk_log2d(x, q, eps, 30), direct.log2d(x, q)) <= 2 * eps
    x, q = dmk_inputs.uniform(2000, seed=4, dim=2)
    assert direct.rel_l2(dmk_log2d(x, q, eps, 40), direct.log2d(x, q)) <= 2 * eps


def test_dmk_log2d_scaling_and_root_leaf():
    x, q = dmk_inputs.uniform(1500, seed=8, dim=2)
    x = 3.0 + 7.0 * x                                  # side 7: -log(7 r) = -log r - log 7
    assert direct.rel_l2(dmk_log2d(x, q, 1e-6, 30), direct.log2d(x, q)) <= 2e-6
    xs, qs = x[:100], q[:100]
    assert np.allclose(dmk_log2d(xs, qs, 1e-6, 200), direct.log2d(xs, qs), rtol=1e-12, atol=1e-12)
