"""Pinned host<->device copy times for the e2e path's buffers (24 MB points, 8 MB
charges H2D, 8 MB potentials D2H) and the plan/eval split of the e2e step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

dev = torch.device("cuda")
for mb in (24, 8):
    h = torch.empty(mb * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
    d = torch.empty_like(h, device=dev)
    for direction in ("h2d", "d2h"):
        ts = []
        for r in range(6):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(f"{direction} {mb} MB: {ms:.3f} ms = {mb * 1.048576 / ms:.1f} GB/s", flush=True)
x, q = dmk_inputs.uniform(1_000_000, seed=1)
Xh, Qh = torch.as_tensor(x).pin_memory(), torch.as_tensor(q).pin_memory()
Uh = torch.empty(1_000_000, dtype=torch.float64).pin_memory()
s = torch.cuda.current_stream()
for r in range(6):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(s)
    plan = dmk.dmk_plan(Xh, eps=1e-6, leaf_capacity=200)
    e1.record(s)
    plan.eval(Qh, out=Uh)
    e2.record(s)
    torch.cuda.synchronize()
    plan.close()
    if r:
        print(f"e2e step: plan(host points) {e0.elapsed_time(e1):.3f} ms, eval(host) {e1.elapsed_time(e2):.3f} ms", flush=True)
