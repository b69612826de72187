"""Serial stage times (DMK_SERIAL=1, DMK_PROFILE=1) of one configuration, plan and eval:
  python scripts/stage_times.py <kind> <n> <eps> <kernel> [reps]"""
import json
import os
import sys
import time

os.environ["DMK_PROFILE"] = "1"
os.environ["DMK_SERIAL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

kind, n, eps, kernel = sys.argv[1], int(float(sys.argv[2])), float(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
x, q = dmk_inputs.make(kind, n, seed=1)
X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
del x, q
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = dmk.dmk_plan(X, eps=eps, leaf_capacity=200, kernel=kernel, lam=10.0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan.eval(Q)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tm = plan.timings()
    plan.close()
    print(json.dumps({"form": os.environ.get("DMK_P2P_FORM", "sym"), "plan_ms": round((t1 - t0) * 1e3, 2),
                      "eval_ms": round((t2 - t1) * 1e3, 2), **{k: round(v, 3) for k, v in tm.items()}}), flush=True)
