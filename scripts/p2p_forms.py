"""Near-field kernel forms side by side: serial stage time of the P2P (DMK_SERIAL=1,
DMK_PROFILE=1, CUDA events), the whole step time, and the near-field difference
between forms, for config 1 and config 2 (and any --cases).

  python scripts/p2p_forms.py [--forms queue,leaf] [--qc 24,32,48]
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

ap = argparse.ArgumentParser()
ap.add_argument("--forms", default="queue,leaf")
ap.add_argument("--qc", default="32")
ap.add_argument("--tc", default="0.08")
ap.add_argument("--cases", default="uniform:1000000:1e-6,clusters:10000000:1e-6")
ap.add_argument("--kernel", default="laplace")
a = ap.parse_args()

for case in a.cases.split(","):
    kind, n, eps = case.split(":")
    n, eps = int(n), float(eps)
    x, q = dmk_inputs.make(kind, n, seed=1)
    X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
    ref = None
    for form in a.forms.split(","):
        for qc, tc in ([(q_, t_) for q_ in a.qc.split(",") for t_ in a.tc.split(",")] if form == "queue"
                       else [("-", "-")]):
            os.environ["DMK_P2P_FORM"] = form
            os.environ["DMK_P2P_QC"] = qc if qc != "-" else "32"
            os.environ["DMK_P2P_TC"] = tc if tc != "-" else "0.08"
            res = {}
            for serial in ("1", "0"):
                os.environ["DMK_SERIAL"] = serial
                ts, steps = [], []
                for rep in range(4):
                    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    s0.record()
                    plan = dmk.dmk_plan(X, eps=eps, leaf_capacity=200, kernel=a.kernel, lam=10.0)
                    plan.eval(Q)
                    s1.record()
                    torch.cuda.synchronize()
                    if rep > 0:
                        steps.append(s0.elapsed_time(s1))
                        ts.append(plan.timings())
                    if serial == "1" and rep == 3:
                        un = plan.stage("unear")
                    plan.close()
                res[serial] = (ts, steps)
            p2p = np.mean([t["p2p"] for t in res["1"][0]])
            d = None
            if ref is None:
                ref = un
            else:
                d = float(np.max(np.abs(un - ref)) / np.max(np.abs(ref)))
            print(json.dumps({"case": case, "form": form, "qc": qc, "tc": tc, "p2p_ms_serial": round(p2p, 4),
                              "step_ms_serial": round(float(np.mean(res["1"][1])), 3),
                              "step_ms_overlap": round(float(np.mean(res["0"][1])), 3),
                              "near_maxrel_vs_first": d}), flush=True)
