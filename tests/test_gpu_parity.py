"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer structure (tree, lists) must match bit for bit; floating-point stages
match the oracle to rounding; potentials match the fp64 direct sum to the
north-star tolerance rel-l2 <= 2 eps.
"""
import numpy as np
import pytest

import dmk_inputs
from oracle import cheb, direct
from oracle.dmk import dmk_laplace3d
from oracle.tree import Tree

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
dmk = pytest.importorskip("paper_2308_00292_b200")


# Stage tolerances per precision tier, about 3x the worst error measured over the three
# cases below (profiles/r02_stage_err_v*.jsonl, scripts/stage_err.py).  p <= 18 (eps 1e-3,
# 1e-6): the fp32 tier of reading R16 (fp32 anterpolation partial sums, fp32-stored
# plane waves, fp32 translation / back transforms / evaluation / P2P pairs), a few fp32
# roundings: measured moments 3.4e-7, outgoing 5.3e-7, local 1.8e-7, far 3.6e-7, near
# 3.2e-7 (max) / 4.1e-7 (l2), total 2.2e-7, linearity 2.7e-7.  p = 28 (eps 1e-9): fp64,
# measured 1.6e-14 / 1.7e-14 / 6.3e-15 / 1.7e-14 / 3.0e-13 / 6.7e-13 / 2.0e-13 / 1.6e-15
# (the near field is bounded by the residual polynomial's fit, 1e-2 eps m0, tables.cu).
TOL = {
    "fp32": dict(moments=1e-6, outgoing=1.5e-6, local=5e-7, ufar=1e-6, near_max=1e-6, near_l2=1.2e-6,
                 total=6e-7, linearity=8e-7),
    "fp64": dict(moments=5e-14, outgoing=5e-14, local=2e-14, ufar=5e-14, near_max=1e-12, near_l2=2e-12,
                 total=6e-13, linearity=5e-15),
}


def tol(p, what):
    return TOL["fp64" if p >= 28 else "fp32"][what]


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def gpu_run(x, q, eps, ns):
    plan = dmk.dmk_plan(cuda(x), eps=eps, leaf_capacity=ns)
    u = plan.eval(cuda(q))
    torch.cuda.synchronize()
    return plan, u.cpu().numpy()


CASES = [("uniform", 10000, 200), ("clusters", 12000, 40), ("sphere", 8000, 60)]
EPS = [1e-3, 1e-6, 1e-9]   # Table 1 rows PAPER.md:2028-2030: p = 9, 18, 28


@pytest.fixture(scope="module", params=[(c, e) for e in EPS for c in CASES],
                ids=[f"{c[0]}-{e:g}" for e in EPS for c in CASES])
def case(request):
    (kind, n, ns), eps = request.param
    x, q = dmk_inputs.make(kind, n, seed=21)
    ref_u, st = dmk_laplace3d(x, q, eps, ns, return_stages=True)
    plan, u = gpu_run(x, q, eps, ns)
    yield dict(x=x, q=q, ns=ns, eps=eps, st=st, T=st["tree"], plan=plan, u=u, ref_u=ref_u)
    plan.close()


def same_points_per_leaf(perm, T):
    """The device's point order: a permutation that puts every leaf's points in the
    leaf's range.  Within a leaf the order is free (the paper fixes none; the device
    sorts by the top 24 Morton bits when the tree ends above level 8, R5)."""
    assert np.array_equal(np.sort(perm), np.arange(len(T.perm)))
    for i in np.nonzero(T.box_leaf)[0]:
        a, b = T.box_start[i], T.box_end[i]
        if not np.array_equal(np.sort(perm[a:b]), np.sort(T.perm[a:b])):
            return False
    return True


def caller_order(sorted_vals, perm):
    """A per-point stage array (sorted order) in the caller's point order."""
    out = np.empty_like(sorted_vals)
    out[perm] = sorted_vals
    return out


def test_tree_bit_exact(case):
    T, plan = case["T"], case["plan"]
    inf = plan.info()
    assert inf.nbox == T.nbox and inf.nlevels == T.nlevels
    assert inf.side == T.side and tuple(inf.lo) == tuple(T.lo)
    assert same_points_per_leaf(plan.tree("perm"), T)
    assert np.array_equal(plan.tree("box_level"), T.box_level)
    assert np.array_equal(plan.tree("box_code"), T.box_code)
    assert np.array_equal(plan.tree("box_start"), T.box_start)
    assert np.array_equal(plan.tree("box_end"), T.box_end)
    assert np.array_equal(plan.tree("box_leaf").astype(bool), T.box_leaf)
    assert np.array_equal(plan.tree("box_parent"), T.box_parent)
    assert np.array_equal(plan.tree("colleagues").reshape(-1, 27), T.box_colleagues)
    assert np.array_equal(plan.tree("fout") >= 0, T.fout)


def test_full_sort_order_bit_exact(monkeypatch):
    """DMK_FULL_SORT=1: the stable sort by the whole 63-bit key (reading R5) -- the device's
    permutation equals the oracle's element by element; the default (top 24 bits first,
    the rest only when a level-7 box needs refinement) gives the same tree."""
    x, q = dmk_inputs.make("sphere", 8000, seed=21)
    T = Tree(x, 60)
    monkeypatch.setenv("DMK_FULL_SORT", "1")
    plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=60)
    perm_full = plan.tree("perm")
    plan.close()
    assert np.array_equal(perm_full, T.perm)
    monkeypatch.delenv("DMK_FULL_SORT")
    plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=60)
    assert np.array_equal(plan.tree("box_code"), T.box_code) and np.array_equal(plan.tree("box_end"), T.box_end)
    assert same_points_per_leaf(plan.tree("perm"), T)
    plan.close()


def test_direct_lists_bit_exact(case):
    T, plan = case["T"], case["plan"]
    off, items = plan.tree("dlist_off"), plan.tree("dlist")
    for i in range(T.nbox):
        assert sorted(items[off[i]:off[i + 1]].tolist()) == T.dlist[i]


def test_moments_match_oracle_proxies(case):
    """Chebyshev moments mu = V^T rho~ (Def. 2.1 with rho~ = V^{-T} mu)."""
    T, plan, st = case["T"], case["plan"], case["st"]
    p = plan.info().p
    mom = plan.stage("moments").reshape(-1, p, p, p)
    Vt = cheb.V(p).T
    fout = plan.tree("fout")
    for i in np.nonzero(T.fout)[0]:
        ref = cheb.apply3([Vt, Vt, Vt], st["proxy"][i])
        got = mom[fout[i]]
        assert np.max(np.abs(got - ref)) <= tol(p, "moments") * max(1.0, np.max(np.abs(ref)))


def phi_from_parity_split(F, nf):
    """Outgoing plane waves Phi(m1, m2, m3), m in [-nf, nf]^3, from the device's real
    parity-split layout F[a][pi][b][c] (kernels.cu):
    Phi(m) = sum_pi i^{|pi|} sgn(m1)^pi1 sgn(m2)^pi2 sgn(m3)^pi3 F_pi[|m1|][|m2|][|m3|]."""
    h = nf + 1
    Fp = F.reshape(h, 8, h, h).transpose(1, 0, 2, 3)
    m = np.arange(-nf, nf + 1)
    am, sg = np.abs(m), np.where(m < 0, -1.0, 1.0)
    out = np.zeros((2 * nf + 1,) * 3, dtype=np.complex128)
    for pi in range(8):
        p1, p2, p3 = (pi >> 2) & 1, (pi >> 1) & 1, pi & 1
        sign = (sg[:, None, None] ** p1) * (sg[None, :, None] ** p2) * (sg[None, None, :] ** p3)
        out += (1j ** (p1 + p2 + p3)) * sign * Fp[pi][np.ix_(am, am, am)]
    return out


def test_outgoing_matches_oracle(case):
    """Outgoing plane waves Phi_l(B) (Eq. 3.42) over the full mode cube, from the device's
    real parity-split representation."""
    T, plan, st = case["T"], case["plan"], case["st"]
    inf = plan.info()
    nf, nf0 = inf.nf, inf.nf0
    s0, s1 = 8 * (nf0 + 1) ** 3, 8 * (nf + 1) ** 3
    phi = plan.stage("outgoing")
    assert phi.size == s0 + (inf.nfout - 1) * s1
    fout = plan.tree("fout")
    for i in np.nonzero(T.fout)[0]:
        r = fout[i]
        if r == 0:
            got = phi_from_parity_split(phi[:s0], nf0)
        else:
            got = phi_from_parity_split(phi[s0 + (r - 1) * s1: s0 + r * s1], nf)
        ref = st["Phi"][i]
        assert np.max(np.abs(got - ref)) <= tol(inf.p, "outgoing") * np.max(np.abs(ref))


def test_local_expansions_match_oracle(case):
    T, plan, st = case["T"], case["plan"], case["st"]
    p = plan.info().p
    lam = plan.stage("local").reshape(-1, p, p, p)
    exp = plan.tree("exp")
    scale = max(np.max(np.abs(st["local"][i])) for i in st["local"])
    for i in np.nonzero(exp >= 0)[0]:
        assert np.max(np.abs(lam[exp[i]] - st["local"][i])) <= tol(p, "local") * scale


def test_far_and_near_fields_match_oracle(case):
    st, plan = case["st"], case["plan"]
    # per-point stages compared in the caller's order (the order within a leaf is free)
    perm, T = plan.tree("perm"), case["T"]
    ufar, unear = caller_order(plan.stage("ufar"), perm), caller_order(plan.stage("unear"), perm)
    p = plan.info().p
    ref_far = caller_order(st["u_far"], T.perm)
    assert np.max(np.abs(ufar - ref_far)) <= tol(p, "ufar") * np.max(np.abs(ref_far))
    # the device evaluates r_L M_L(r) through a polynomial fitted to 1e-2 eps m0
    # (tables.cu); the oracle uses the exact Legendre series.  p <= 18:
    # pairs in fp32 on double-single leaf-local coordinates (reading R16)
    ref_near = caller_order(st["u_near"] + st["u_self"], T.perm)
    assert np.max(np.abs(unear - ref_near)) <= tol(p, "near_max") * np.max(np.abs(ref_near))
    assert np.linalg.norm(unear - ref_near) <= tol(p, "near_l2") * np.linalg.norm(ref_near)


def test_potential_matches_oracle_dmk_and_direct(case):
    u, ref_u = case["u"], case["ref_u"]
    assert np.max(np.abs(u - ref_u)) <= tol(case["plan"].info().p, "total") * np.max(np.abs(ref_u))
    ref = direct.laplace3d(case["x"], case["q"])
    assert direct.rel_l2(u, ref) <= 2 * case["eps"]


def test_linearity_per_tier(case):
    """u(q1) + u(q2) = u(q1 + q2) on one plan, to the tier's roundings."""
    plan, q1 = case["plan"], case["q"]
    q2 = np.random.default_rng(10).uniform(-1, 1, q1.shape[0])
    # q1 last: the plan's stage buffers end as they were (the other tests read them)
    b, c, a = (plan.eval(cuda(v)).cpu().numpy() for v in (q2, q1 + q2, q1))
    assert np.max(np.abs(a + b - c)) <= tol(plan.info().p, "linearity") * np.max(np.abs(c))


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_config0_all_precisions(eps):
    """BASELINE config 0: N = 10,000 uniform in [0,1]^3, charges U[-1,1], n_s = 200."""
    x, q = dmk_inputs.uniform(10000, seed=0)
    ref = direct.laplace3d(x, q)
    plan, u = gpu_run(x, q, eps, 200)
    plan.close()
    assert direct.rel_l2(u, ref) <= 2 * eps


@pytest.mark.parametrize("kind,n,ns", [("clusters", 30000, 50), ("sphere", 30000, 100)])
def test_adaptive_distributions_vs_direct(kind, n, ns):
    x, q = dmk_inputs.make(kind, n, seed=5)
    ref = direct.laplace3d(x, q)
    plan, u = gpu_run(x, q, 1e-6, ns)
    plan.close()
    assert direct.rel_l2(u, ref) <= 2e-6


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_config1_full_size_sampled(eps):
    """BASELINE config 1 at full size (N = 1e6, n_s = 200, the launch the bench times) at
    every precision tier of Table 1: the oracle direct sum at 400
    sampled targets, rel-l2 <= 2 eps."""
    x, q = dmk_inputs.uniform(1_000_000, seed=1)
    plan, u = gpu_run(x, q, eps, 200)
    plan.close()
    idx = np.random.default_rng(2).choice(x.shape[0], 400, replace=False)
    ref = np.array([np.sum(np.delete(q, i) / np.linalg.norm(np.delete(x, i, axis=0) - x[i], axis=1))
                    for i in idx])
    assert direct.rel_l2(u[idx], ref) <= 2 * eps


def test_root_leaf_exact():
    x, q = dmk_inputs.uniform(150, seed=3)
    plan, u = gpu_run(x, q, 1e-6, 200)
    plan.close()
    assert np.allclose(u, direct.laplace3d(x, q), rtol=1e-12, atol=0)


def test_degenerate_points():
    # one point; two points; duplicated points (coincident pairs omitted)
    plan, u = gpu_run(np.array([[0.3, 0.2, 0.1]]), np.array([2.0]), 1e-6, 200)
    plan.close()
    assert u[0] == 0.0
    x = np.array([[0.0, 0.0, 0.0], [3.0, 4.0, 0.0]])
    plan, u = gpu_run(x, np.array([1.0, 2.0]), 1e-6, 1)
    plan.close()
    assert direct.rel_l2(u, [2.0 / 5.0, 1.0 / 5.0]) <= 2e-6
    xb, qb = dmk_inputs.uniform(3000, seed=4)
    x = np.concatenate([xb, xb[:500]])
    q = np.concatenate([qb, qb[:500] * 0.5])
    plan, u = gpu_run(x, q, 1e-6, 40)
    plan.close()
    assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2e-6
    # all points identical: every pair is coincident, the exact potential is 0.
    # Below n_s the root is a leaf and the result is exactly 0.  Above n_s the tree
    # refines to LMAX and the far field's self terms cancel against -M_L(0) rho
    # (Step 5) only to eps * M_LMAX(0) * sum|rho| -- the method's bound (R9).
    x = np.tile([[0.5, 0.5, 0.5]], (300, 1))
    plan, u = gpu_run(x, np.ones(300), 1e-6, 400)
    plan.close()
    assert np.all(u == 0.0)
    plan, u = gpu_run(x, np.ones(300), 1e-6, 50)
    info = plan.info()
    plan.close()
    m_lmax0 = 2.0 ** (info.nlevels - 1) * 3.0        # ~ psi(0)/(c0 r_L)
    assert info.nlevels == 21 and np.all(np.isfinite(u))
    assert np.max(np.abs(u)) <= 10 * 1e-6 * m_lmax0 * 300


def test_deterministic_and_host_path():
    x, q = dmk_inputs.clusters(20000, seed=8)
    plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=60)
    a = plan.eval(cuda(q)).cpu().numpy()
    b = plan.eval(cuda(q)).cpu().numpy()
    h = plan.eval(np.asarray(q))            # host buffers: H2D + D2H inside the call
    plan.close()
    assert np.array_equal(a, b) and np.array_equal(a, h)
    plan_h = dmk.dmk_plan(x, eps=1e-6, leaf_capacity=60)      # host points
    assert np.array_equal(plan_h.eval(np.asarray(q)), a)
    plan_h.close()


def test_linearity():
    x, q1 = dmk_inputs.uniform(20000, seed=9)
    q2 = np.random.default_rng(10).uniform(-1, 1, x.shape[0])
    plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=100)
    a, b, c = (plan.eval(cuda(v)).cpu().numpy() for v in (q1, q2, q1 + q2))
    plan.close()
    assert np.max(np.abs(a + b - c)) <= tol(18, "linearity") * np.max(np.abs(c))


@pytest.mark.parametrize("kernel", ["laplace", "yukawa"])
def test_p2p_forms_agree(kernel, monkeypatch):
    """The four fp32-tier near-field kernels: the symmetric form (default, k_p2p32s:
    same-level leaf pairs evaluated once for both leaves, mixed-level entries by the
    queue form), the queue form (k_p2p32q, DMK_P2P_FORM=queue), the per-pair form
    (k_p2p32, DMK_P2P_FORM=leaf) and the Sec. 3.4 form (octant work items, source octants
    culled by their distance to the target octant, PAPER.md:1362-1391,
    DMK_P2P_FORM=octant) against each other and the direct sum: culled pairs have
    r >= r_L where R_L = 0 (1/r; Yukawa culls r >= r_L in every form, reading R13), so the
    forms agree to fp32 summation order.  The clustered input has leaves at many levels,
    so every form's mixed-level entries are exercised."""
    x, q = dmk_inputs.clusters(30000, seed=31)
    lam = 10.0 if kernel == "yukawa" else 0.0
    res = {}
    for form in ("sym", "queue", "leaf", "octant"):
        monkeypatch.setenv("DMK_P2P_FORM", form)
        plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=200, kernel=kernel, lam=lam)
        u = plan.eval(cuda(q)).cpu().numpy()
        res[form] = (u, plan.stage("unear"))
        plan.close()
    ref = direct.yukawa3d(x, q, lam) if kernel == "yukawa" else direct.laplace3d(x, q)
    nl = res["leaf"][1]
    for form in ("sym", "queue", "octant"):
        u, nf = res[form]
        assert np.max(np.abs(nf - nl)) <= 1e-6 * np.max(np.abs(nl)), form
        assert direct.rel_l2(u, ref) <= 2e-6, form


@pytest.mark.parametrize("kernel", ["laplace", "yukawa"])
@pytest.mark.parametrize("cap", [20, 50, 300])
def test_p2p_symmetric_chunks(kernel, cap, monkeypatch):
    """The symmetric form evaluates the same-level leaf pairs in chunks of 32 points per
    leaf (the larger chunk on the lanes, the other broadcast): leaf capacities 20, 50 and
    300 give single chunks, 2-chunk leaves and leaves of up to 10 chunks, on a uniform
    cloud (all entries same-level) and on clusters (mixed levels: the queue form takes
    the list suffixes).  The near field equals the per-pair form's to fp32 summation
    order and the potential is within 2 eps of the direct sum at sampled targets."""
    lam = 10.0 if kernel == "yukawa" else 0.0
    for kind in ("uniform", "clusters"):
        x, q = dmk_inputs.make(kind, 40000, seed=34)
        res = {}
        for form in ("sym", "leaf"):
            monkeypatch.setenv("DMK_P2P_FORM", form)
            plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=cap, kernel=kernel, lam=lam)
            u = plan.eval(cuda(q)).cpu().numpy()
            res[form] = (u, plan.stage("unear"))
            plan.close()
        nl = res["leaf"][1]
        assert np.max(np.abs(res["sym"][1] - nl)) <= 1e-6 * np.max(np.abs(nl)), kind
        idx = np.random.default_rng(3).choice(x.shape[0], 300, replace=False)
        ref = (direct.yukawa3d(x, q, lam, targets=x[idx]) if kernel == "yukawa"
               else direct.laplace3d(x, q, targets=x[idx]))
        assert direct.rel_l2(res["sym"][0][idx], ref) <= 2e-6, kind


@pytest.mark.parametrize("qc", ["24", "32", "48"])
def test_p2p_queue_capacities(qc, monkeypatch):
    """The queue form drains whenever a lane's queue nears capacity: every capacity gives
    the same near field (clustered leaves of 200 points fill the queues many times per
    item), to fp32 summation order."""
    x, q = dmk_inputs.clusters(20000, seed=32)
    out = {}
    for c in ("32", qc):
        monkeypatch.setenv("DMK_P2P_QC", c)
        plan = dmk.dmk_plan(cuda(x), eps=1e-6, leaf_capacity=200)
        plan.eval(cuda(q))
        out[c] = plan.stage("unear")
        plan.close()
    assert np.max(np.abs(out[qc] - out["32"])) <= 1e-6 * np.max(np.abs(out["32"]))


@pytest.mark.parametrize("eps", [1e-3, 1e-6])
def test_anterp_tensor_core_form(eps, monkeypatch):
    """Anterpolation on the 5th-generation tensor cores (tcgen05 kind::tf32, 3xTF32 split,
    warp-specialised: producer warps write the operands of 8-point chunks into two shared
    buffers, one MMA warp issues; TMEM accumulators flushed to fp64 every 64 points;
    DMK_ANTERP=tc) against the oracle's proxy charges (Def. 2.1, mu = V^T rho~) on a deep
    adaptive tree.  The 3xTF32 products carry ~2^-21 relative error and the fp32 sums run
    over 64 points: measured 1.1e-6 (profiles/r02_anterp_forms_v6.jsonl)."""
    monkeypatch.setenv("DMK_ANTERP", "tc")
    x, q = dmk_inputs.make("clusters", 12000, seed=21)
    _, st = dmk_laplace3d(x, q, eps, 40, return_stages=True)
    T = st["tree"]
    plan, u = gpu_run(x, q, eps, 40)
    p = plan.info().p
    mom = plan.stage("moments").reshape(-1, p, p, p)
    fout = plan.tree("fout")
    plan.close()
    Vt = cheb.V(p).T
    for i in np.nonzero(T.fout)[0]:
        ref = cheb.apply3([Vt, Vt, Vt], st["proxy"][i])
        assert np.max(np.abs(mom[fout[i]] - ref)) <= 2e-6 * max(1.0, np.max(np.abs(ref)))
    assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2 * eps


@pytest.mark.parametrize("eps", [1e-3, 1e-6])
def test_eval_forms_agree(eps, monkeypatch):
    """Far-field evaluation on the tensor cores (default, k_eval_tc: tcgen05 kind::tf32,
    3xTF32) and on packed FFMA2 (DMK_EVAL=ffma, k_eval32): both against the oracle's far
    field (Step 3 leaf evaluation) on a deep adaptive tree."""
    x, q = dmk_inputs.make("sphere", 8000, seed=21)
    _, st = dmk_laplace3d(x, q, eps, 60, return_stages=True)
    for form in ("tc", "ffma"):
        monkeypatch.setenv("DMK_EVAL", form)
        plan, u = gpu_run(x, q, eps, 60)
        ufar = caller_order(plan.stage("ufar"), plan.tree("perm"))
        plan.close()
        ref_far = caller_order(st["u_far"], st["tree"].perm)
        assert np.max(np.abs(ufar - ref_far)) <= tol(18, "ufar") * np.max(np.abs(ref_far)), form
        assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2 * eps, form


def test_pw64_parent_group_form(monkeypatch):
    """eps = 1e-9 (p = 28, fp64): the parent-group translation (k_pwshift64: the 8 children
    of a parent from the 4x4x4 window of outgoing expansions, Eq. 3.39, then the back
    transforms from T, Eqs. 3.43-3.44; DMK_PW64=group) against the oracle's local
    expansions and the default per-box form."""
    x, q = dmk_inputs.make("sphere", 8000, seed=21)
    _, st = dmk_laplace3d(x, q, 1e-9, 60, return_stages=True)
    res = {}
    for form in ("group", "staged", "box"):
        monkeypatch.setenv("DMK_PW64", form)
        plan, u = gpu_run(x, q, 1e-9, 60)
        p = plan.info().p
        lam = plan.stage("local").reshape(-1, p, p, p)
        ex = plan.tree("exp")
        plan.close()
        scale = max(np.max(np.abs(st["local"][i])) for i in st["local"])
        for i in np.nonzero(ex >= 0)[0]:
            assert np.max(np.abs(lam[ex[i]] - st["local"][i])) <= tol(28, "local") * scale, form
        res[form] = u
    for form in ("group", "staged"):
        assert np.max(np.abs(res[form] - res["box"])) <= 1e-13 * np.max(np.abs(res["box"])), form
        assert direct.rel_l2(res[form], direct.laplace3d(x, q)) <= 2e-9, form


@pytest.mark.parametrize("kind,n,ns", [("sphere", 8000, 60), ("clusters", 12000, 40)])
def test_prox2pw64_forms(monkeypatch, kind, n, ns):
    """eps = 1e-9 (p = 28): T_prox2pw (Eq. 3.42) by the register-blocked DMMA sweeps
    (default) and by the independent-tile form (DMK_PROX2PW=tiles): both against the
    oracle's outgoing expansions over the full mode cube, and against each other (the
    same products in the same k order: the stored parity-split arrays agree to rounding)."""
    x, q = dmk_inputs.make(kind, n, seed=23)
    _, st = dmk_laplace3d(x, q, 1e-9, ns, return_stages=True)
    T = st["tree"]
    raw = {}
    for form in ("sweep", "tiles"):
        monkeypatch.setenv("DMK_PROX2PW", form)
        plan, u = gpu_run(x, q, 1e-9, ns)
        inf = plan.info()
        nf, nf0 = inf.nf, inf.nf0
        s0, s1 = 8 * (nf0 + 1) ** 3, 8 * (nf + 1) ** 3
        phi = plan.stage("outgoing")
        fout = plan.tree("fout")
        plan.close()
        assert phi.size == s0 + (inf.nfout - 1) * s1
        for i in np.nonzero(T.fout)[0][:40]:
            r = fout[i]
            got = phi_from_parity_split(phi[:s0], nf0) if r == 0 else \
                phi_from_parity_split(phi[s0 + (r - 1) * s1: s0 + r * s1], nf)
            ref = st["Phi"][i]
            assert np.max(np.abs(got - ref)) <= tol(28, "outgoing") * np.max(np.abs(ref)), form
        raw[form] = phi
        assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2e-9, form
    assert np.max(np.abs(raw["sweep"] - raw["tiles"])) <= 1e-13 * np.max(np.abs(raw["tiles"]))


@pytest.mark.parametrize("kind,n,ns", [("clusters", 12000, 40), ("uniform", 20000, 60)])
def test_pw64_staged_deep(monkeypatch, kind, n, ns):
    """The staged parent-group translation (k_pwshift_s<H, double>: Z, Y, X window passes
    through shared memory) + DMMA back transforms (k_pw2poly64) on deeper trees (clustered:
    ~11 levels, missing window boxes; uniform 2e4 at n_s = 60: full 4x4x4 windows) against
    the oracle's local expansions (Eq. 3.39, Eqs. 3.43-3.44) and the direct sum."""
    monkeypatch.setenv("DMK_PW64", "staged")
    x, q = dmk_inputs.make(kind, n, seed=23)
    _, st = dmk_laplace3d(x, q, 1e-9, ns, return_stages=True)
    plan, u = gpu_run(x, q, 1e-9, ns)
    p = plan.info().p
    lam = plan.stage("local").reshape(-1, p, p, p)
    ex = plan.tree("exp")
    plan.close()
    scale = max(np.max(np.abs(st["local"][i])) for i in st["local"])
    for i in np.nonzero(ex >= 0)[0]:
        assert np.max(np.abs(lam[ex[i]] - st["local"][i])) <= tol(28, "local") * scale
    assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2e-9


@pytest.mark.parametrize("eps", [1e-3, 1e-6])
@pytest.mark.parametrize("kind,n,ns", [("clusters", 12000, 40), ("sphere", 8000, 60)])
def test_pws_staged_fp32_tier(monkeypatch, eps, kind, n, ns):
    """fp32 tier (R16): the staged translation (k_pwshift_s<H, float>, DMK_PWS=staged)
    against the oracle's local expansions and the register form (k_pwshift)."""
    x, q = dmk_inputs.make(kind, n, seed=24)
    _, st = dmk_laplace3d(x, q, eps, ns, return_stages=True)
    lams = {}
    for form in ("staged", "reg"):
        monkeypatch.setenv("DMK_PWS", form)
        plan, u = gpu_run(x, q, eps, ns)
        p = plan.info().p
        lam = plan.stage("local").reshape(-1, p, p, p)
        ex = plan.tree("exp")
        plan.close()
        scale = max(np.max(np.abs(st["local"][i])) for i in st["local"])
        for i in np.nonzero(ex >= 0)[0]:
            assert np.max(np.abs(lam[ex[i]] - st["local"][i])) <= tol(p, "local") * scale, form
        assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2 * eps, form
        lams[form] = lam
    assert np.max(np.abs(lams["staged"] - lams["reg"])) <= 2e-7 * np.max(np.abs(lams["reg"]))
