"""Plan (tree) phase timings and eval stage timings at config 1 (DMK_PROFILE_TREE=1,
DMK_SERIAL=1): synchronising marks, for finding where plan time goes."""
import os
import sys

os.environ["DMK_PROFILE"] = "1"
os.environ["DMK_PROFILE_TREE"] = "1"
os.environ["DMK_SERIAL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
kind = sys.argv[2] if len(sys.argv) > 2 else "uniform"
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
x, q = dmk_inputs.make(kind, n, seed=1)
X = torch.as_tensor(x, device="cuda")
Q = torch.as_tensor(q, device="cuda")
for r in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = dmk.dmk_plan(X, eps=eps, leaf_capacity=200)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan.eval(Q)
    torch.cuda.synchronize()
    tm = plan.timings()
    plan.close()
    if r >= 2:
        print(f"plan {1e3 * (t1 - t0):.3f} ms: " + ", ".join(f"{k} {v:.3f}" for k, v in tm.items()), flush=True)
