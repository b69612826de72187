"""One DMK step (plan + eval) repeated --reps times at config-1 size, for ncu runs.

  python scripts/prof_step.py [--n 1000000] [--eps 1e-6] [--ns 200] [--reps 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--eps", type=float, default=1e-6)
ap.add_argument("--ns", type=int, default=200)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kind", default="uniform")
ap.add_argument("--kernel", default="laplace")
ap.add_argument("--lam", type=float, default=10.0)
a = ap.parse_args()
x, q = dmk_inputs.make(a.kind, a.n, seed=1)
X = torch.as_tensor(x, device="cuda")
Q = torch.as_tensor(q, device="cuda")
for r in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = dmk.dmk_plan(X, eps=a.eps, leaf_capacity=a.ns, kernel=a.kernel, lam=a.lam)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    u = plan.eval(Q)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tm = plan.timings()
    inf = plan.info()
    plan.close()
    print(f"rep {r}: plan {1e3 * (t1 - t0):.2f} ms  eval {1e3 * (t2 - t1):.2f} ms  nbox {inf.nbox} "
          f"levels {inf.nlevels}  {', '.join(f'{k} {v:.3f}' for k, v in tm.items())}", flush=True)
