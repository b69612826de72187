"""One small DMK evaluation (the near field is what is of interest) for debugging runs:
  python scripts/p2p_small.py [kind] [n] [leaf_capacity] [kernel]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 200
kernel = sys.argv[4] if len(sys.argv) > 4 else "laplace"
x, q = dmk_inputs.make(kind, n, seed=1)
plan = dmk.dmk_plan(torch.as_tensor(x, device="cuda"), eps=1e-6, leaf_capacity=cap, kernel=kernel, lam=10.0)
u = plan.eval(torch.as_tensor(q, device="cuda"))
torch.cuda.synchronize()
un = plan.stage("unear")
plan.close()
print(kind, n, cap, kernel, "unear max", float(np.max(np.abs(un))), flush=True)
