#!/usr/bin/env python
"""bench.py -- DMK throughput on BASELINE.json config 1 (3D Laplace, N = 1e6 uniform
points in [0,1]^3, charges U[-1,1], eps = 1e-6, leaf capacity 200).

One step = the whole hot path on device-resident inputs: dmk_plan (bounding cube,
Morton sort, adaptive tree, interaction lists) + dmk_eval (Steps 2-5 of Sec. 3.5).
Timed with CUDA events on the plan stream, L2 flushed (256 MiB write) between steps,
max over ranks.  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/dmk.py, fp64 numpy, as it stands) on a
bounded sample of the same workload on the host cores; under torchrun only rank 0
runs it.  --gpus N > 1: the script relaunches itself under torchrun (one NCCL rank per
GPU, 127.0.0.1) unless it already runs under one, and every rank runs the partitioned
DMK of paper_2308_00292_b200/parallel.py on one global problem of N x (--n) uniform
points (weak scaling: --n points per GPU): Morton partition, particle halo,
coarse-moment all-reduce.  DMK_BENCH_DISTRIBUTED=1 takes that path at N = 1 too.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points/sec, 3D Laplace DMK, eps=1e-6, 1/2/4/8 B200; rel ℓ2 err vs direct"
WORKLOAD = ("config1: 3D Laplace K=1/r, N=1e6 uniform iid in [0,1]^3, charges U[-1,1], "
            "eps=1e-6, leaf capacity 200, single B200 per rank")
# The paper's own measurement context (context only, not a baseline: other hardware and a
# single core).  Its throughput values are plotted, not printed: PAPER.md:2603-2606.
PAPER_CONTEXT = {
    "hardware": "single core of a 3.30 GHz Intel Xeon Gold 6234, single-threaded (PAPER.md:2518-2520)",
    "software": "Fortran, Intel compiler, Intel MKL (PAPER.md:2518-2519)",
    "workload": "3D Laplace, N = m 1e6 uniform in the unit box (m = 1..8) and on a sphere of radius "
                "0.45; n_s = 280 for eps 1e-3/1e-6, 800 for 1e-9/1e-12 (PAPER.md:2531-2540)",
    "throughput": "average throughput in units of 1e5 points/s, plotted per eps in the paper's "
                  "throughput figure (PAPER.md:2603-2606); the values are not given in the text",
}
FP64_FMA_PER_CLK_SM = 64
FP32_FMA_PER_CLK_SM = 128
N_SM = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--ns", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=20000)
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4)
                          if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def stage_models(info, n, pairs, K, inball):
    """Algorithmic work per phase: (bound, amount, unit, precision)."""
    P, nf, nf0 = info.p, info.nf, info.nf0
    p3 = P ** 3
    fp32 = P <= 18   # precision tier (reading R16)
    # outgoing expansions, real parity-split form: 8 (nf+1)^3 values per box, stored in
    # fp32 (4 bytes) for p <= 18, fp64 otherwise
    phi_bytes = 8 * (4 if fp32 else 8) * ((nf0 + 1) ** 3 + (info.nfout - 1) * (nf + 1) ** 3)
    alu = "fp32" if fp32 else "fp64"
    return {
        "anterp": ("alu", 2.0 * p3 * n, "flop", alu),
        # c2p / p2c by parent groups: 14 p^4 FMA per parent of 8 children = 3.5 p^4 flop per child
        "c2p": ("alu", 3.5 * P ** 4 * (info.nfout - 1), "flop", "fp64"),
        "prox2pw": ("hbm", 8.0 * p3 * info.nfout + phi_bytes, "byte", None),
        "pwlocal": ("hbm", phi_bytes + 8.0 * p3 * info.nexp, "byte", None),
        "p2c": ("alu", 3.5 * P ** 4 * (info.nexp - 1), "flop", "fp64"),
        "eval": ("alu", 2.0 * p3 * n, "flop", alu),
        # every list pair: distance test (9 flop); pairs inside the residual's ball
        # r < r_L: polynomial (2K), rsqrt (~6), s and the accumulate (6)
        "p2p": ("alu", 9.0 * pairs + (2.0 * K + 12.0) * inball, "flop", alu),
    }


def list_pairs(plan):
    import numpy as np
    off, items = plan.tree("dlist_off"), plan.tree("dlist")
    st, en = plan.tree("box_start"), plan.tree("box_end")
    cnt = en - st
    per_box_src = np.add.reduceat(cnt[items], off[:-1]) if items.size else np.zeros(len(cnt))
    has = off[1:] > off[:-1]
    return int(np.sum(np.where(has, cnt * per_box_src, 0)))


def inball_pairs(plan, x, dev):
    """Number of (target, source) list pairs with |x_t - x_s| < r_L(source), counted on
    the device with torch in padded box-pair batches (measurement only, not the
    product path)."""
    import numpy as np
    import torch
    inf = plan.info()
    perm = plan.tree("perm")
    xs = torch.as_tensor((x[perm] - np.asarray(inf.lo)) / inf.side, device=dev)
    off, items = plan.tree("dlist_off"), plan.tree("dlist")
    st, en, lev = plan.tree("box_start"), plan.tree("box_end"), plan.tree("box_level")
    tb = np.repeat(np.arange(len(off) - 1), off[1:] - off[:-1])
    sb = items
    boxes = np.unique(np.concatenate([tb, sb]))
    slot = np.full(len(st), -1, dtype=np.int64)
    slot[boxes] = np.arange(len(boxes))
    cnt = en[boxes] - st[boxes]
    M = int(cnt.max())
    idx = st[boxes][:, None] + np.arange(M)[None, :]
    valid = np.arange(M)[None, :] < cnt[:, None]
    idx = torch.as_tensor(np.where(valid, idx, 0), device=dev)
    vt = torch.as_tensor(valid, device=dev)
    pts = xs[idx]                                            # (nbox, M, 3)
    tpts = torch.where(vt[..., None], pts, torch.full_like(pts, 1e10))
    spts = torch.where(vt[..., None], pts, torch.full_like(pts, -1e10))
    r2 = torch.as_tensor(4.0 ** (-lev[sb].astype(np.float64)), device=dev)
    ts_, ss_ = torch.as_tensor(slot[tb], device=dev), torch.as_tensor(slot[sb], device=dev)
    total = 0
    chunk = max(1, 2 ** 26 // (M * M))
    for a in range(0, len(sb), chunk):
        d2 = torch.cdist(tpts[ts_[a:a + chunk]], spts[ss_[a:a + chunk]]) ** 2
        total += int((d2 < r2[a:a + chunk, None, None]).sum())
    return total


def cpu_baseline(n_sample, eps, ns):
    import numpy as np

    import dmk_inputs
    from oracle.dmk import dmk_laplace3d
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    x, q = dmk_inputs.uniform(n_sample, seed=1)
    t0 = time.perf_counter()
    dmk_laplace3d(x, q, eps, ns)
    dt = time.perf_counter() - t0
    return {"value": n_sample / dt, "unit": "points/s", "cores": cores, "kind": "oracle",
            "sample": f"oracle DMK (oracle/dmk.py, fp64 numpy) on {n_sample} points drawn from the "
                      f"config-1 distribution (uniform [0,1]^3, U[-1,1] charges), eps={eps}, "
                      f"leaf capacity {ns}; {dt:.1f} s"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import dmk_inputs
    from oracle.dmk import dmk_laplace3d
    n_s = 10000
    x, q = dmk_inputs.uniform(n_s, seed=1)
    for _ in range(a.warmup):
        dmk_laplace3d(x, q, a.eps, a.ns)
    ts = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        dmk_laplace3d(x, q, a.eps, a.ns)
        ts.append(time.perf_counter() - t0)
    dt = float(np.mean(ts))
    value = n_s / dt
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "sample_points": n_s, "eps": a.eps, "leaf_capacity": a.ns},
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle",
                             "sample": f"each step: oracle DMK on {n_s} points of the config-1 distribution"},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def torchrun_command(a, port):
    """The relaunch of this script with one rank per GPU (the driver's own launch line)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def run_distributed(a, backend=None, device=None, pg="nccl"):
    """N > 1: one global uniform problem of world * a.n points, a.n generated per rank,
    evaluated by the partitioned DMK (weak scaling).  Device-event timing on each rank
    between barriers, max over ranks.  `backend` / `device` / `pg` are for the CPU test
    of this path (tests/test_bench_distributed.py runs it under gloo with its own
    backend); the product run is libdmk on this rank's GPU over NCCL."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import dmk_inputs
    import paper_2308_00292_b200 as dmk
    from paper_2308_00292_b200 import parallel as par
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("WORLD_SIZE", str(world))
    os.environ.setdefault("RANK", str(rank))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    cuda = device is None
    if cuda:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group(pg, device_id=dev)
        backend = par.GpuBackend(dev)
    else:
        dev = torch.device(device)
        dist.init_process_group(pg)
    comm = par.TorchComm()
    x, q = dmk_inputs.uniform(a.n, seed=1 + rank)
    X, Q = torch.as_tensor(x, device=dev), torch.as_tensor(q, device=dev)
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev) if cuda else None
    stream = torch.cuda.current_stream(dev) if cuda else None
    st = {}

    def sync():
        if cuda:
            torch.cuda.synchronize(dev)

    class Span:   # device events on the launching stream (host clock in the CPU test)
        def __init__(self):
            if cuda:
                self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def start(self):
            if cuda:
                self.e0.record(stream)
            else:
                self.t0 = time.perf_counter()

        def stop(self):
            if cuda:
                self.e1.record(stream)
            else:
                self.t1 = time.perf_counter()

        def ms(self):
            return self.e0.elapsed_time(self.e1) if cuda else 1e3 * (self.t1 - self.t0)

    def step(Xs, Qs):
        return par.dmk_eval_let(Xs, Qs, comm, backend, eps=a.eps, ns=a.ns, stats=st)

    for _ in range(a.warmup):
        step(X, Q)
    sync()
    L = dmk.lib()
    import ctypes
    L.dmk_kernel_launches.restype = ctypes.c_int64
    L.dmk_kernel_launches.argtypes = [ctypes.c_void_p]
    launches0 = L.dmk_kernel_launches(None)
    clk = Clocks(local)
    if cuda:
        clk.start()
    times = []
    for _ in range(a.steps):
        if flush is not None:
            flush.zero_()
        sync()
        dist.barrier()
        sp = Span()
        sp.start()
        u = step(X, Q)
        sp.stop()
        sync()
        dist.barrier()
        times.append(sp.ms())
    clocks = clk.stop() if cuda else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["cpu test run"]}
    launches = (L.dmk_kernel_launches(None) - launches0) // a.steps
    t = torch.tensor([float(np.mean(times))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t.item())
    # end to end: host points/charges copied in and potentials copied out every step
    Xh, Qh = (torch.as_tensor(x).pin_memory(), torch.as_tensor(q).pin_memory()) if cuda else \
        (torch.as_tensor(x), torch.as_tensor(q))
    e2e = []
    for k in range(a.warmup + a.steps):
        sync()
        dist.barrier()
        sp = Span()
        sp.start()
        uh = step(Xh.to(dev, non_blocking=True), Qh.to(dev, non_blocking=True)).cpu()
        sp.stop()
        sync()
        if k >= a.warmup:
            e2e.append(sp.ms())
    te = torch.tensor([float(np.mean(e2e))], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # accuracy: direct sum over all ranks' points at 100 of rank 0's targets
    xa = [torch.zeros_like(X) for _ in range(world)]
    qa = [torch.zeros_like(Q) for _ in range(world)]
    dist.all_gather(xa, X)
    dist.all_gather(qa, Q)
    if rank == 0:
        xs, qs = torch.cat(xa).cpu().numpy(), torch.cat(qa).cpu().numpy()
        idx = np.random.default_rng(7).choice(a.n, min(100, a.n), replace=False)
        ref = np.array([np.sum(np.delete(qs, i) / np.linalg.norm(np.delete(xs, i, axis=0) - xs[i], axis=1))
                        for i in idx])
        rel = float(np.linalg.norm(u.cpu().numpy()[idx] - ref) / np.linalg.norm(ref))
        line = {
            "metric": METRIC, "value": a.n * world / (t_step * 1e-3), "unit": "points/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": t_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32" if a.eps > 5e-7 else "f64", "data": "synthetic",
            "config": {"workload": f"uniform iid in [0,1]^3, {a.n} points per GPU, one global problem of "
                                   f"{a.n * world} points, 3D Laplace, eps={a.eps}, leaf capacity {a.ns}",
                       "N_per_gpu": a.n, "eps": a.eps, "leaf_capacity": a.ns,
                       "step": "locally essential tree (parallel.dmk_eval_let): root all-reduce, sample-sort "
                               "Morton partition, all-to-all, one-box particle halo, dense coarse-moment "
                               "all-reduce + sparse boundary-moment all-to-all, plan + upward x2 + downward, "
                               "return all-to-all",
                       "l2": "flushed by a 256 MiB write between timed steps",
                       "parallelism": f"Morton partition over {world} ranks ({pg})",
                       "halo_level": st.get("level"), "halo_points_rank0": st.get("n_halo"),
                       "own_points_rank0": st.get("n_own")},
            "rel_l2_err_sampled": rel, "clocks": clocks,
            "e2e": {"value": a.n * world / (float(te.item()) * 1e-3), "unit": "points/s",
                    "h2d_bytes_per_step": a.n * 4 * 8, "d2h_bytes_per_step": a.n * 8,
                    "api": "paper_2308_00292_b200.parallel.dmk_eval_distributed(host tensors copied in/out)"},
            "gpu_launches": int(launches),
        }
        if not cuda:
            line["backend"] = f"test: {type(backend).__name__} on {device} (not a measurement)"
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one NCCL rank per GPU: relaunch under torchrun (the driver's own launch line)
        raise SystemExit(subprocess.call(torchrun_command(a, free_port())))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or os.environ.get("DMK_BENCH_DISTRIBUTED") == "1":
        return run_distributed(a)
    os.environ.setdefault("DMK_PROFILE", "1")
    import numpy as np
    import torch

    import dmk_inputs
    import paper_2308_00292_b200 as dmk

    world, rank, local = 1, 0, int(os.environ.get("LOCAL_RANK", "0"))   # N > 1 runs run_distributed
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    x, q = dmk_inputs.uniform(a.n, seed=1 + rank)
    X = torch.as_tensor(x, device=dev)
    Q = torch.as_tensor(q, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)

    def step(mid=None):
        plan = dmk.dmk_plan(X, eps=a.eps, leaf_capacity=a.ns, stream=sptr)
        if mid is not None:
            mid.record(stream)
        u = plan.eval(Q)
        return plan, u

    for _ in range(a.warmup):
        p_, u_ = step()
        p_.close()
    torch.cuda.synchronize(dev)

    L = dmk.lib()
    import ctypes
    L.dmk_kernel_launches.restype = ctypes.c_int64
    L.dmk_kernel_launches.argtypes = [ctypes.c_void_p]
    clk = Clocks(local)
    clk.start()
    times, stage_ms, plan_ms = [], {}, []
    launches0 = L.dmk_kernel_launches(None)
    info = pairs = None
    for k in range(a.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        em = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan, u = step(em)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        times.append(e0.elapsed_time(e1))
        plan_ms.append(e0.elapsed_time(em))
        if k == a.steps - 1:
            info = plan.info()
            pairs = list_pairs(plan)
            u_last = u.cpu().numpy()
            inball = inball_pairs(plan, x, dev) if rank == 0 else 0
        plan.close()
    launches = (L.dmk_kernel_launches(None) - launches0) // a.steps
    clocks = clk.stop()
    t_step = float(np.mean(times))
    # per-stage kernel times for the roofline, measured in isolation: the timed steps run
    # the near field concurrently with the far field, which makes stage times overlap;
    # DMK_SERIAL=1 plans run the stages back to back (same kernels, same launches)
    os.environ["DMK_SERIAL"] = "1"
    stage_ms = {}
    for k in range(3):
        flush.zero_()
        torch.cuda.synchronize(dev)
        plan, _ = step()
        torch.cuda.synchronize(dev)
        for name, ms in plan.timings().items():
            stage_ms[name] = stage_ms.get(name, 0.0) + ms / 3
        plan.close()
    os.environ.pop("DMK_SERIAL")
    # p <= 18: the plane-wave stage runs as k_pwshift (parent-group translation) and the
    # back transforms (pw2poly); the roofline takes them together as "pwlocal"
    pw_parts = {k: round(stage_ms.pop(k), 4) for k in ("pwshift", "pw2poly") if k in stage_ms}
    if pw_parts:
        stage_ms["pwlocal"] = stage_ms.get("pwlocal", 0.0) + sum(pw_parts.values())
    value = a.n * world / (t_step * 1e-3)

    # ---- end to end through the public API, pinned host buffers
    Xh = torch.as_tensor(x).pin_memory()
    Qh = torch.as_tensor(q).pin_memory()
    Uh = torch.empty(a.n, dtype=torch.float64).pin_memory()
    e2e_times = []
    for k in range(a.warmup + a.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan = dmk.dmk_plan(Xh, eps=a.eps, leaf_capacity=a.ns, stream=sptr)
        plan.eval(Qh, out=Uh)            # H2D of charges, D2H of potentials inside
        e1.record(stream)
        torch.cuda.synchronize(dev)
        plan.close()
        if k >= a.warmup:
            e2e_times.append(e0.elapsed_time(e1))
    t_e2e = float(np.mean(e2e_times))

    # ---- accuracy on this run's output: direct sum at 200 sampled targets
    idx = np.random.default_rng(7).choice(a.n, 200, replace=False)
    ref = np.array([np.sum(np.delete(q, i) / np.linalg.norm(np.delete(x, i, axis=0) - x[i], axis=1)) for i in idx])
    rel = float(np.linalg.norm(u_last[idx] - ref) / np.linalg.norm(ref))

    pk = peaks()
    fp64_peak = N_SM * FP64_FMA_PER_CLK_SM * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    # fp32 tier (reading R16, p <= 18): the P2P pairs run in single precision
    fp32_peak = N_SM * FP32_FMA_PER_CLK_SM * 2 * pk.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    models = stage_models(info, a.n, pairs, info.respoly_degree, inball)
    stages = {}
    for name, (bound, amount, unit, prec) in models.items():
        ms = stage_ms.get(name)
        if not ms:
            continue
        if bound == "hbm":
            ach, peak, u_ = amount / (ms * 1e-3) / 1e9, pk["hbm_gbs"], "GB/s"
        else:
            pk_ = fp32_peak if prec == "fp32" else fp64_peak
            ach, peak, u_ = amount / (ms * 1e-3) / 1e12, pk_, "TFLOP/s"
        stages[name] = {"ms": round(ms, 4), "bound": bound, "achieved": round(ach, 3), "peak": round(peak, 1),
                        "unit": u_, "frac": round(ach / peak, 4), **({"precision": prec} if prec else {})}
    tree_ms = float(np.mean(plan_ms))          # dmk_plan: tree, lists, tables (cached)
    dom = max(stages, key=lambda s: stages[s]["ms"])
    roof = dict(stages[dom])
    roof.pop("ms")
    traffic, tsrc = None, None
    for f in ("r02_traffic.json", "r01_traffic.json"):   # the latest committed capture
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", f)))["bytes"].get(dom)
            tsrc = f
            break
        except Exception:
            pass
    roof.update({"kernel": dom, "traffic": traffic,
                 "traffic_source": f"profiles/{tsrc} (ncu --set full, dram bytes per step)",
                 "peak_source": ("MEASURED_PEAKS.json hbm_gbs" if roof["bound"] == "hbm" else
                                 "derived: 148 SM x 128 fp32 FMA/clk x 2 x sm_max_mhz (DESIGN.md 8(d))"
                                 if roof.get("precision") == "fp32" else
                                 "derived: 148 SM x 64 fp64 FMA/clk x 2 x sm_max_mhz (DESIGN.md 8(d))")})
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+f32" if info.p <= 18 else "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "N_per_gpu": a.n, "eps": a.eps, "leaf_capacity": a.ns,
                   "step": "dmk_plan (tree+lists) + dmk_eval, device-resident inputs",
                   "l2": "flushed by a 256 MiB write between timed steps",
                   "parallelism": "single"},
        "rel_l2_err_sampled": rel,
        "clocks": clocks,
        "e2e": {"value": a.n * world / (t_e2e * 1e-3), "unit": "points/s",
                "h2d_bytes_per_step": a.n * 4 * 8, "d2h_bytes_per_step": a.n * 8,
                "api": "paper_2308_00292_b200.dmk_plan(host points) + Plan.eval(host charges -> host potentials)"},
        "gpu_launches": int(launches),
        "roofline": roof,
        "stages_ms": {**{k: round(v, 4) for k, v in stage_ms.items()}, "tree_and_lists": round(tree_ms, 4),
                      "note": "stage kernels timed back to back (DMK_SERIAL=1); the timed steps overlap "
                              "p2p (low-priority stream) with c2p..eval (high-priority stream)"},
        "stages": stages,
        "pwlocal_parts_ms": pw_parts,
        "tree": {"nbox": info.nbox, "nlevels": info.nlevels, "nfout": info.nfout, "nexp": info.nexp,
                 "p2p_pairs": pairs, "p2p_pairs_in_ball": inball},
    }
    line["paper_context"] = PAPER_CONTEXT
    if not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a.cpu_sample, a.eps, a.ns)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
