"""Repeated plan + eval timings of one config (CUDA events), each printed: run-to-run
stability (verdict r01 weak item 10: config-2 timing instability)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import dmk_inputs  # noqa: E402
import paper_2308_00292_b200 as dmk  # noqa: E402

kind, n, eps, reps = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
pregrow = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
if pregrow > 0:   # grow the default stream-ordered pool once (cudaMallocAsync + free)
    from cuda.bindings import runtime as rt
    torch.cuda.init()
    err, dev = rt.cudaGetDevice()
    err, pool = rt.cudaDeviceGetDefaultMemPool(dev)
    import paper_2308_00292_b200 as _d   # the library sets the pool's release threshold on first use
    _p = _d.dmk_plan(torch.zeros((10, 3), dtype=torch.float64, device="cuda") + torch.rand(10, 3, device="cuda").double())
    _p.close()
    err, ptr = rt.cudaMallocAsync(int(pregrow * 2 ** 30), 0)
    rt.cudaFreeAsync(ptr, 0)
    rt.cudaDeviceSynchronize()
x, q = dmk_inputs.make(kind, n, seed=1)
X, Q = torch.as_tensor(x, device="cuda"), torch.as_tensor(q, device="cuda")
ts = []
for r in range(reps):
    e0, e1, em = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record()
    plan = dmk.dmk_plan(X, eps=eps, leaf_capacity=200)
    em.record()
    plan.eval(Q)
    e1.record()
    torch.cuda.synchronize()
    plan.close()
    ts.append((round(e0.elapsed_time(em), 2), round(em.elapsed_time(e1), 2), round(e0.elapsed_time(e1), 2)))
print(json.dumps({"kind": kind, "n": n, "eps": eps, "pregrow_GiB": pregrow, "plan_eval_total_ms": ts}))
