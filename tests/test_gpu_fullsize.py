"""BASELINE configs 2 and 4 at full size on one B200, checked against the fp64 direct sum
(oracle) at sampled targets (rel-l2 <= 2 eps), plus the tree depth config 2 asks for."""
import numpy as np
import pytest

import dmk_inputs
from oracle import direct

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
dmk = pytest.importorskip("paper_2308_00292_b200")


def sampled_direct(x, q, idx, kernel, lam=0.0):
    f = direct.laplace3d if kernel == "laplace" else (lambda *a, **k: direct.yukawa3d(*a, lam=lam, **k))
    return np.concatenate([f(x, q, targets=x[i:i + 1], chunk=1) for i in idx])


def test_config2_clustered_1e7():
    """Config 2: N = 1e7, 90% in 10 Gaussian clusters (sigma 1e-3..1e-2) + 10% uniform,
    N(0,1) charges, eps = 1e-6.  The config's "depth >= 15" is not reachable with n_s =
    200 for sigma >= 1e-3 (a 9e5-point cluster of sigma 1e-3 holds > 200 points per box
    only down to level ~13; DESIGN.md input recipe): we check the deep adaptive tree the
    recipe does produce (>= 12 levels below the root)."""
    x, q = dmk_inputs.clusters(10_000_000, seed=2)
    X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
    plan = dmk.dmk_plan(X, eps=1e-6, leaf_capacity=200)
    u = plan.eval(Q).cpu().numpy()
    depth = plan.info().nlevels - 1
    plan.close()
    assert depth >= 12
    idx = np.random.default_rng(4).choice(len(x), 200, replace=False)
    assert direct.rel_l2(u[idx], sampled_direct(x, q, idx, "laplace")) <= 2e-6


def test_config4_yukawa_1e8_single_gpu():
    """Config 4's problem on one GPU: N = 1e8 uniform, K = exp(-10 r)/r, eps = 1e-6."""
    x, q = dmk_inputs.uniform(100_000_000, seed=3)
    X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
    del x
    plan = dmk.dmk_plan(X, eps=1e-6, leaf_capacity=200, kernel="yukawa", lam=10.0)
    u = plan.eval(Q).cpu().numpy()
    plan.close()
    idx = np.random.default_rng(5).choice(len(q), 32, replace=False)
    x = X.cpu().numpy()
    del X, Q
    torch.cuda.empty_cache()
    assert direct.rel_l2(u[idx], sampled_direct(x, q, idx, "yukawa", 10.0)) <= 2e-6
