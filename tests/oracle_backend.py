"""Oracle-backed backend for the distributed driver (test infrastructure only): the same
four calls as paper_2308_00292_b200.parallel.GpuBackend, computed by oracle/dmk.py with
its root / min_level / level_get / level_set hooks.  Dense level data are the oracle's
proxy charges (the device exchanges Chebyshev moments; both are linear in the charges,
which is all the all-reduce needs)."""
import numpy as np
import torch

from oracle.dmk import dmk


class OracleBackend:
    def plan(self, points, eps, ns, kernel, lam, root, min_level, n_targets=0):
        return {"x": points.cpu().numpy(), "eps": eps, "ns": ns, "kernel": kernel, "lam": lam, "root": list(root) if root is not None else None,
                "min_level": min_level}

    def upward(self, plan, charges):
        plan["q"] = charges.cpu().numpy()

    def _run(self, plan, **kw):
        return dmk(plan["x"], plan["q"], plan["eps"], plan["ns"], plan["kernel"], plan["lam"], root=plan["root"],
                   min_level=plan["min_level"], **kw)

    def get_level(self, plan, level):
        return torch.as_tensor(self._run(plan, level_get=level))

    def set_level(self, plan, level, dense):
        plan["set"] = (level, dense.cpu().numpy())

    def get_boxes(self, plan, level, codes):
        return torch.as_tensor(self._run(plan, box_get=(level, [int(c) for c in codes])))

    def set_boxes(self, plan, level, codes, values):
        plan.setdefault("bset", []).append((level, [int(c) for c in codes], values.cpu().numpy()))

    def downward(self, plan):
        return torch.as_tensor(self._run(plan, level_set=plan.get("set"), box_set=plan.get("bset")))

    def close(self, plan):
        pass
