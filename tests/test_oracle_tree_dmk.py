"""Pins for oracle/tree.py (Sec. 3.2 / 3.5 Step 0) and oracle/dmk.py (Sec. 3.5)."""
import numpy as np
import pytest

import dmk_inputs
from oracle import direct
from oracle.dmk import dmk_laplace3d
from oracle.kernels import LaplaceSplit
from oracle.params import for_eps
from oracle.tree import LMAX, NBITS, Tree, morton3


def brute_morton(q):
    out = []
    for row in q:
        k = 0
        for b in range(NBITS):
            for d in range(3):
                if (int(row[d]) >> b) & 1:
                    k |= 1 << (3 * b + (2 - d))
        out.append(k)
    return np.array(out, dtype=np.int64)


def boxes_touch(T, i, j):
    """Closed boxes share a point."""
    si, sj = 2.0 ** -T.box_level[i], 2.0 ** -T.box_level[j]
    li, lj = T.box_coords[i] * si, T.box_coords[j] * sj
    return bool(np.all((li <= lj + sj) & (lj <= li + si)))


def box_gap(T, i, j, ord=2):
    """Distance between closed boxes i and j (Euclidean, or sup-norm for ord=inf)."""
    si, sj = 2.0 ** -T.box_level[i], 2.0 ** -T.box_level[j]
    li, lj = T.box_coords[i] * si, T.box_coords[j] * sj
    g = np.maximum(0, np.maximum(li - (lj + sj), lj - (li + si)))
    return float(np.linalg.norm(g, ord=ord))


def test_morton_matches_bitwise_definition():
    rng = np.random.default_rng(0)
    q = rng.integers(0, 2 ** NBITS, (200, 3))
    assert np.array_equal(morton3(q), brute_morton(q))


def test_eight_octant_points():
    """One point per octant, n_s = 1: a single split, 8 leaves at level 1."""
    x = np.array([[a, b, c] for a in (0.25, 0.75) for b in (0.25, 0.75) for c in (0.25, 0.75)])
    T = Tree(x, 1)
    assert T.nbox == 9 and T.nlevels == 2
    assert np.sum(T.box_leaf) == 8 and np.all(T.box_npts[1:] == 1)


@pytest.fixture(scope="module", params=["uniform", "clusters", "sphere"])
def tree(request):
    x, _ = dmk_inputs.make(request.param, 3000, seed=7)
    return Tree(x, 20)


def test_partition_and_capacity(tree):
    T = tree
    leaves = np.nonzero(T.box_leaf & (T.box_npts > 0))[0]
    cover = np.zeros(T.N, dtype=int)
    for i in leaves:
        cover[T.box_start[i]:T.box_end[i]] += 1
        assert T.box_npts[i] <= T.ns or T.box_level[i] == LMAX
        c, s = T.center(i), 2.0 ** -T.box_level[i]
        assert np.all(np.abs(T.xs[T.box_start[i]:T.box_end[i]] - c) <= s / 2 + 1e-15)
    assert np.all(cover == 1)


def test_level_restriction_exhaustive(tree):
    """No two touching leaves differ by more than one level."""
    T = tree
    leaves = np.nonzero(T.box_leaf)[0]
    for a in range(len(leaves)):
        for b in range(a + 1, len(leaves)):
            i, j = leaves[a], leaves[b]
            if abs(int(T.box_level[i]) - int(T.box_level[j])) > 1:
                assert not boxes_touch(T, i, j)


def test_colleagues_brute_force(tree):
    T = tree
    for i in range(T.nbox):
        same = [j for j in range(T.level_offset[T.box_level[i]], T.level_offset[T.box_level[i] + 1])
                if boxes_touch(T, i, j)]
        assert sorted(same) == sorted(int(s) for s in T.box_colleagues[i] if s >= 0)


def test_direct_lists_complete(tree):
    """Every (target leaf B, source leaf S) pair whose boxes come within r_{L_S}
    (the residual support, Eq. 3.66) is in B's list; listed pairs are within the
    colleague geometry."""
    T = tree
    leaves = [i for i in np.nonzero(T.box_leaf & (T.box_npts > 0))[0]]
    for b in leaves:
        lst = set(T.dlist[b])
        for s in leaves:
            if box_gap(T, b, s) < 2.0 ** -T.box_level[s]:
                assert s in lst
        for s in lst:
            assert box_gap(T, b, s, np.inf) <= 2.0 ** -min(T.box_level[s], T.box_level[b])


def test_flags_and_pw_lists(tree):
    T = tree
    for i in range(T.nbox):
        assert T.fout[i] == ((not T.box_leaf[i]) and T.box_npts[i] > 0)
        if T.box_npts[i] > 0:
            want = [int(s) for s in T.box_colleagues[i] if s >= 0 and T.fout[s]]
            assert T.pwlist[i] == want
            assert T.fin[i] == (len(want) > 0)


# ---------------------------------------------------------------------------- DMK
@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_dmk_uniform_matches_direct(eps):
    x, q = dmk_inputs.uniform(3000, seed=11)
    ref = direct.laplace3d(x, q)
    u = dmk_laplace3d(x, q, eps, 100)
    assert direct.rel_l2(u, ref) <= 2 * eps


@pytest.mark.parametrize("kind", ["clusters", "sphere"])
def test_dmk_adaptive_matches_direct(kind):
    x, q = dmk_inputs.make(kind, 3000, seed=12)
    ref = direct.laplace3d(x, q)
    u = dmk_laplace3d(x, q, 1e-6, 30)
    assert direct.rel_l2(u, ref) <= 2e-6


def test_dmk_root_leaf_is_exact():
    x, q = dmk_inputs.uniform(150, seed=13)
    u = dmk_laplace3d(x, q, 1e-6, 200)
    assert np.allclose(u, direct.laplace3d(x, q), rtol=1e-13, atol=0)


def test_dmk_stage_decomposition():
    """u_far = sum_j M_{L_j}(x_i - y_j) rho_j (far field of every source through its
    own leaf level, Eq. 3.47) and u_near = sum over the lists of R_{L_j} (Eq. 3.48)."""
    x, q = dmk_inputs.clusters(2000, seed=14)
    u, st = dmk_laplace3d(x, q, 1e-6, 30, return_stages=True)
    T = st["tree"]
    S = LaplaceSplit(for_eps(1e-6).c)
    X, rho = T.xs, q[T.perm]
    Ls = T.box_level[T.point_leaf]
    d = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    far, near = np.zeros(T.N), np.zeros(T.N)
    for L in np.unique(Ls):
        cols = Ls == L
        far += S.M(int(L), d[:, cols]) @ rho[cols]
        dd = d[:, cols]
        near += np.where(dd > 0, S.R(int(L), np.where(dd > 0, dd, 1.0)), 0.0) @ rho[cols]
    assert np.linalg.norm(st["u_far"] - far) <= 1e-6 * np.linalg.norm(far)
    assert np.max(np.abs(st["u_near"] - near)) <= 1e-12 * np.max(np.abs(near))
    assert np.allclose(st["u_self"], -rho * S.M0_at_zero(1) * 2.0 ** (Ls - 1), rtol=1e-14)


def test_dmk_linearity_and_determinism():
    x, q1 = dmk_inputs.uniform(1500, seed=15)
    q2 = np.random.default_rng(16).uniform(-1, 1, 1500)
    a = dmk_laplace3d(x, q1, 1e-3, 60)
    b = dmk_laplace3d(x, q2, 1e-3, 60)
    c = dmk_laplace3d(x, q1 + q2, 1e-3, 60)
    assert np.max(np.abs(a + b - c)) < 1e-12 * np.max(np.abs(c))
    assert np.array_equal(a, dmk_laplace3d(x, q1, 1e-3, 60))
