"""Time dmk_plan + dmk_eval (device-resident inputs, CUDA events) for the BASELINE configs
on one GPU and print one JSON line per config.  Not the bench contract: a record of the
other configs' single-GPU throughput for profiles/.

  python scripts/configs_timing.py [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", default="")
a = ap.parse_args()
CONFIGS = [
    ("config0 laplace uniform 1e4 eps1e-6", "uniform", 10_000, 1e-6, "laplace", 0.0),
    ("config1 laplace uniform 1e6 eps1e-3", "uniform", 1_000_000, 1e-3, "laplace", 0.0),
    ("config1 laplace uniform 1e6 eps1e-6", "uniform", 1_000_000, 1e-6, "laplace", 0.0),
    ("config1 laplace uniform 1e6 eps1e-9", "uniform", 1_000_000, 1e-9, "laplace", 0.0),
    ("config2 laplace clusters 1e7 eps1e-6", "clusters", 10_000_000, 1e-6, "laplace", 0.0),
    ("config3 log2d circle 1e7 eps1e-9", "circle2d", 10_000_000, 1e-9, "log", 0.0),
    ("config4 yukawa uniform 1e8 eps1e-6 (1 GPU)", "uniform", 100_000_000, 1e-6, "yukawa", 10.0),
]
for name, kind, n, eps, kernel, lam in CONFIGS:
    if a.only and not any(o in name for o in a.only.split("|")):
        continue
    x, q = dmk_inputs.make(kind, n, seed=1)
    X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
    del x, q
    ts = []
    for r in range(a.reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan = dmk.dmk_plan(X, eps=eps, leaf_capacity=200, kernel=kernel, lam=lam)
        plan.eval(Q)
        e1.record()
        torch.cuda.synchronize()
        inf = plan.info()
        plan.close()
        if r:
            ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    print(json.dumps({"config": name, "n": n, "ms_per_step": round(ms, 3), "points_per_s": n / (ms * 1e-3),
                      "levels": inf.nlevels, "nbox": inf.nbox, "p": inf.p}), flush=True)
    del X, Q
    torch.cuda.empty_cache()
