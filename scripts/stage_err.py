"""Measured stage-by-stage error of the device path against the oracle, per precision
tier and case (the quantities tests/test_gpu_parity.py bounds), to set the stage
tolerances from measurement (about 3x the worst measured value).  Also config 1 at
N = 1e6 against the sampled direct sum for every eps.  Prints one JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402
from oracle import cheb, direct  # noqa: E402
from oracle.dmk import dmk_laplace3d  # noqa: E402


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def phi_from_parity_split(F, nf):
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


def stage_errors(kind, n, ns, eps):
    x, q = dmk_inputs.make(kind, n, seed=21)
    ref_u, st = dmk_laplace3d(x, q, eps, ns, return_stages=True)
    T = st["tree"]
    plan = dmk.dmk_plan(cuda(x), eps=eps, leaf_capacity=ns)
    u = plan.eval(cuda(q)).cpu().numpy()
    inf = plan.info()
    p, nf, nf0 = inf.p, inf.nf, inf.nf0
    fout = plan.tree("fout")
    mom = plan.stage("moments").reshape(-1, p, p, p)
    Vt = cheb.V(p).T
    e_mom = 0.0
    for i in np.nonzero(T.fout)[0]:
        ref = cheb.apply3([Vt, Vt, Vt], st["proxy"][i])
        e_mom = max(e_mom, np.max(np.abs(mom[fout[i]] - ref)) / max(1.0, np.max(np.abs(ref))))
    s0, s1 = 8 * (nf0 + 1) ** 3, 8 * (nf + 1) ** 3
    phi = plan.stage("outgoing")
    e_phi = 0.0
    for i in np.nonzero(T.fout)[0]:
        r = fout[i]
        got = phi_from_parity_split(phi[:s0], nf0) if r == 0 else \
            phi_from_parity_split(phi[s0 + (r - 1) * s1: s0 + r * s1], nf)
        ref = st["Phi"][i]
        e_phi = max(e_phi, np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    lam = plan.stage("local").reshape(-1, p, p, p)
    ex = plan.tree("exp")
    scale = max(np.max(np.abs(st["local"][i])) for i in st["local"])
    e_loc = max(np.max(np.abs(lam[ex[i]] - st["local"][i])) for i in np.nonzero(ex >= 0)[0]) / scale
    def caller(v, perm):
        out = np.empty_like(v)
        out[perm] = v
        return out
    dperm = plan.tree("perm")
    ufar, unear = caller(plan.stage("ufar"), dperm), caller(plan.stage("unear"), dperm)
    ref_far = caller(st["u_far"], T.perm)
    e_far = np.max(np.abs(ufar - ref_far)) / np.max(np.abs(ref_far))
    ref_near = caller(st["u_near"] + st["u_self"], T.perm)
    e_near_max = np.max(np.abs(unear - ref_near)) / np.max(np.abs(ref_near))
    e_near_l2 = np.linalg.norm(unear - ref_near) / np.linalg.norm(ref_near)
    e_tot_oracle = np.max(np.abs(u - ref_u)) / np.max(np.abs(ref_u))
    e_direct = direct.rel_l2(u, direct.laplace3d(x, q))
    q2 = np.random.default_rng(10).uniform(-1, 1, n)
    b = plan.eval(cuda(q2)).cpu().numpy()
    c = plan.eval(cuda(q + q2)).cpu().numpy()
    e_lin = np.max(np.abs(u + b - c)) / np.max(np.abs(c))
    plan.close()
    return dict(kind=kind, n=n, ns=ns, eps=eps, p=p, nlevels=int(inf.nlevels), moments=e_mom, outgoing=e_phi,
                local=e_loc, ufar=e_far, near_max=e_near_max, near_l2=e_near_l2, total_vs_oracle=e_tot_oracle,
                vs_direct=e_direct, linearity=e_lin)


def config1(eps, nsamp=400):
    x, q = dmk_inputs.uniform(1_000_000, seed=1)
    plan = dmk.dmk_plan(cuda(x), eps=eps, leaf_capacity=200)
    u = plan.eval(cuda(q)).cpu().numpy()
    plan.close()
    idx = np.random.default_rng(2).choice(x.shape[0], nsamp, replace=False)
    ref = np.array([np.sum(np.delete(q, i) / np.linalg.norm(np.delete(x, i, axis=0) - x[i], axis=1)) for i in idx])
    return dict(config=1, eps=eps, n=1_000_000, samples=nsamp, rel_l2=direct.rel_l2(u[idx], ref))


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "stages"):
        for eps in (1e-3, 1e-6, 1e-9):
            for kind, n, ns in [("uniform", 10000, 200), ("clusters", 12000, 40), ("sphere", 8000, 60)]:
                print(json.dumps(stage_errors(kind, n, ns, eps)), flush=True)
    if which in ("all", "config1"):
        for eps in (1e-3, 1e-6, 1e-9):
            print(json.dumps(config1(eps)), flush=True)
