"""Near-field (P2P) error of the device against the oracle's stage values, per case:
max and l2 relative errors, and the whole potential against the direct sum."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402
from oracle import direct  # noqa: E402
from oracle.dmk import dmk_laplace3d  # noqa: E402

for kind, n, ns, eps in [("uniform", 10000, 200, 1e-6), ("clusters", 12000, 40, 1e-6), ("sphere", 8000, 60, 1e-6),
                         ("uniform", 10000, 200, 1e-3), ("clusters", 12000, 40, 1e-3)]:
    x, q = dmk_inputs.make(kind, n, seed=21)
    ref_u, st = dmk_laplace3d(x, q, eps, ns, return_stages=True)
    plan = dmk.dmk_plan(torch.as_tensor(x, device="cuda"), eps=eps, leaf_capacity=ns)
    u = plan.eval(torch.as_tensor(q, device="cuda")).cpu().numpy()
    unear = plan.stage("unear")
    plan.close()
    ref = st["u_near"] + st["u_self"]
    d = unear - ref
    print(f"{kind} n={n} ns={ns} eps={eps}: near max rel {np.max(np.abs(d)) / np.max(np.abs(ref)):.2e} "
          f"l2 rel {np.linalg.norm(d) / np.linalg.norm(ref):.2e}  total vs direct "
          f"{direct.rel_l2(u, direct.laplace3d(x, q)):.2e}", flush=True)
