"""The distributed DMK path on the device: dmk_upward / dmk_level_moments / dmk_downward
through the C ABI, and paper_2308_00292_b200.parallel with thread ranks sharing one B200
(the host exchanges meet at a barrier; no kernel waits on another rank)."""
import numpy as np
import pytest

import dmk_inputs
from oracle import direct

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
dmk = pytest.importorskip("paper_2308_00292_b200")
from paper_2308_00292_b200 import parallel as par  # noqa: E402


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def test_split_eval_equals_eval_and_level_roundtrip():
    x, q = dmk_inputs.uniform(30000, seed=3)
    lo = x.min(0)
    side = float((x.max(0) - lo).max())
    plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=60, root=list(lo) + [side], min_level=3)
    a = plan.eval(cuda(q)).cpu().numpy()
    plan.upward(cuda(q))
    dense = plan.level_moments(2, torch.empty((64,) + (plan.info().p,) * 3, dtype=torch.float64, device="cuda"))
    plan.level_moments(2, dense.clone(), set=True)     # set(get) rebuilds the same coarse levels
    b = plan.downward(device="cuda").cpu().numpy()
    plan.close()
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))
    assert direct.rel_l2(a, direct.laplace3d(x, q)) <= 2e-6


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("kernel", ["laplace", "yukawa"])
def test_thread_ranks_on_one_gpu(world, kernel):
    x, q = dmk_inputs.clusters(40000, seed=9)
    who = np.random.default_rng(world).integers(0, world, len(x))
    lam = 10.0 if kernel == "yukawa" else 0.0

    def fn(comm):
        m = who == comm.rank
        st = {}
        u = par.dmk_eval_distributed(cuda(x[m]), cuda(q[m]), comm, par.GpuBackend("cuda"), eps=1e-6, ns=80,
                                     kernel=kernel, lam=lam, stats=st)
        torch.cuda.synchronize()
        return u.cpu().numpy(), st

    res = par.run_threads(world, fn)
    u = np.empty(len(x))
    for r in range(world):
        u[who == r] = res[r][0]
    assert sum(r[1]["n_own"] for r in res) == len(x)
    ref = direct.laplace3d(x, q) if kernel == "laplace" else direct.yukawa3d(x, q, lam)
    assert direct.rel_l2(u, ref) <= 2e-6


def test_n_targets_restricts_work_not_results():
    """dmk_options.n_targets: only the first t caller points are targets (a distributed
    rank's own points ahead of its halo).  Their potentials are bit-identical to those of
    a plan in which every point is a target; fewer local expansions and P2P items run."""
    x, q = dmk_inputs.uniform(60000, seed=12)
    order = np.argsort(x[:, 0], kind="stable")     # targets: the half with x < median, first
    x, q = x[order], q[order]
    t = 30000
    full = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=80)
    a = full.eval(cuda(q)).cpu().numpy()
    nexp_full = full.info().nexp
    full.close()
    part = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=80, n_targets=t)
    b = part.eval(cuda(q)).cpu().numpy()
    nexp_part = part.info().nexp
    part.close()
    assert np.array_equal(a[:t], b[:t])
    assert nexp_part < nexp_full


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kernel", ["laplace", "yukawa"])
def test_let_thread_ranks_on_one_gpu(world, kernel):
    """The locally-essential-tree evaluation (parallel.dmk_eval_let: sample-sort ownership,
    one-box particle halo, dense + sparse boundary moment exchange through
    dmk_level_moments / dmk_box_moments) on the device, thread ranks sharing one B200."""
    x, q = dmk_inputs.clusters(40000, seed=9)
    who = np.random.default_rng(world).integers(0, world, len(x))
    lam = 10.0 if kernel == "yukawa" else 0.0

    def fn(comm):
        m = who == comm.rank
        st = {}
        u = par.dmk_eval_let(cuda(x[m]), cuda(q[m]), comm, par.GpuBackend("cuda"), eps=1e-6, ns=80, kernel=kernel,
                             lam=lam, levels=3, stats=st)
        torch.cuda.synchronize()
        return u.cpu().numpy(), st

    res = par.run_threads(world, fn)
    u = np.empty(len(x))
    for r in range(world):
        u[who == r] = res[r][0]
    assert sum(r[1]["n_own"] for r in res) == len(x)
    ref = direct.laplace3d(x, q) if kernel == "laplace" else direct.yukawa3d(x, q, lam)
    assert direct.rel_l2(u, ref) <= 2e-6


def test_box_moments_roundtrip():
    """dmk_box_moments reads and writes the listed boxes of a forced level without touching
    the others; set(get) leaves the evaluation unchanged."""
    x, q = dmk_inputs.uniform(30000, seed=3)
    lo = x.min(0)
    side = float((x.max(0) - lo).max())
    plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=60, root=list(lo) + [side], min_level=3)
    a = plan.eval(cuda(q)).cpu().numpy()
    plan.upward(cuda(q))
    p = plan.info().p
    dense = plan.level_moments(2, torch.empty((64, p, p, p), dtype=torch.float64, device="cuda"))
    codes = np.array([5, 17, 63, 0])
    vals = plan.box_moments(2, codes)
    assert np.array_equal(vals, dense.cpu().numpy()[codes])
    plan.box_moments(2, codes, vals, set=True)
    b = plan.downward(device="cuda").cpu().numpy()
    plan.close()
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(a))
