"""Compare kernel forms selected by an environment variable (e.g. DMK_ANTERP=ffma|tc):
serial stage times at config 1 (DMK_SERIAL=1, DMK_PROFILE=1, CUDA events) and the
stage-by-stage error against the oracle on the parity cases (scripts/stage_err.py).

  python scripts/stage_forms.py DMK_ANTERP ffma,tc [--eps 1e-6,1e-3] [--kinds uniform,clusters,sphere]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DMK_PROFILE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402
from scripts.stage_err import stage_errors  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("var")
ap.add_argument("values")
ap.add_argument("--eps", default="1e-6,1e-3")
ap.add_argument("--kinds", default="uniform,clusters,sphere")
ap.add_argument("--no-err", action="store_true")
a = ap.parse_args()
CASES = {"uniform": (10000, 200), "clusters": (12000, 40), "sphere": (8000, 60)}
x, q = dmk_inputs.uniform(1_000_000, seed=1)
X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
for v in a.values.split(","):
    os.environ[a.var] = v
    for eps in [float(e) for e in a.eps.split(",")]:
        os.environ["DMK_SERIAL"] = "1"
        tms = []
        for rep in range(4):
            plan = dmk.dmk_plan(X, eps=eps, leaf_capacity=200)
            plan.eval(Q)
            torch.cuda.synchronize()
            if rep:
                tms.append(plan.timings())
            plan.close()
        os.environ.pop("DMK_SERIAL")
        st = {k: round(float(np.mean([t[k] for t in tms])), 4) for k in tms[0]}
        print(json.dumps({a.var: v, "eps": eps, "config1_serial_ms": st}), flush=True)
        if a.no_err:
            continue
        for kind in a.kinds.split(","):
            n, ns = CASES[kind]
            print(json.dumps({a.var: v, **stage_errors(kind, n, ns, eps)}), flush=True)
