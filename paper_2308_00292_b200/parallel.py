"""Distributed DMK evaluation: one process (or thread) per GPU, points partitioned along
the Morton curve (BASELINE config 4; DESIGN.md §8 row a9).

Decomposition (per rank r; all device work through the C ABI of libdmk, the exchanges
through a Comm -- NCCL/gloo via torch.distributed, or in-process threads):

  1. root box   all-reduce MIN/MAX of the local coordinates -> the single-process root
                cube of reading R5 (lo = min, side = max extent), shared by all ranks.
  2. partition  every point's box at level Lc (its Morton code, computed exactly as the
                library does: q = floor((x - lo) * 2^21/side)); all-reduce SUM of the
                level-Lc histogram; contiguous Morton ranges of level-(Lc-1) boxes with
                balanced point counts -> owner(box) (an Lc-box belongs to its parent's
                owner, so every level-(Lc-1) box lies on one rank).
  3. exchange   all-to-all: each point goes to the owner of its Lc-box.
  4. halo       all-to-all: each owned point also goes to every rank owning a colleague
                of its Lc-box (the neighbour-halo particles).  Every colleague, at any
                level >= Lc, of an owned box lies inside own + halo boxes, and every pair
                whose Lc-ancestors are not colleagues interacts only through the levels
                < Lc (the difference kernels D_l, l >= Lc, vanish beyond r_l).
  5. local plan dmk_plan over own + halo points with the shared root and min_level = Lc
                (levels < Lc forced dense, so every rank has the same coarse boxes).
  6. coarse     dmk_upward with all local charges; the moments of the OWNED level-(Lc-1)
                boxes are exact (all their points are own points), the others are zeroed
                (dmk_level_moments get); all-reduce SUM -> the global coarse moments (the
                replicated coarse levels of the north star).
  7. local      dmk_level_moments set (level Lc-1 and the c2p rebuild of the levels
                above), dmk_downward -> potentials of own + halo points; the own ones are
                kept.
  8. return     all-to-all of the potentials back to the ranks/indices the points came from.

The halo is one Lc-box thick; the ghost work it costs is the price of this first
decomposition (the locally-essential-tree refinement -- exchanging boundary moments /
plane waves instead of whole Lc-boxes -- is the next step).

Backends: GpuBackend (the product: libdmk on the rank's CUDA device).  The CPU gloo
tests plug an oracle-backed backend in through the same four calls.
"""
from __future__ import annotations

import functools
import math
import threading
from typing import List, Sequence

import numpy as np
import torch

NBITS = 21


# ---------------------------------------------------------------- communicators
class Comm:
    rank: int
    world: int

    def allreduce(self, t: torch.Tensor, op: str) -> torch.Tensor:   # op in {"sum", "min", "max"}
        raise NotImplementedError

    def alltoallv(self, sends: List[torch.Tensor]) -> List[torch.Tensor]:
        """sends[d] (float64 [k_d, w]) goes to rank d; returns the list received from each rank."""
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed process group (NCCL over NVLink on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce(self, t, op):
        ops = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX}
        t = t.clone()
        self.dist.all_reduce(t, op=ops[op], group=self.group)
        return t

    def alltoallv(self, sends):
        w = sends[0].shape[1]
        dev = sends[0].device
        cnt = torch.tensor([s.shape[0] for s in sends], dtype=torch.int64, device=dev)
        rcnt = torch.empty_like(cnt)
        self.dist.all_to_all_single(rcnt, cnt, group=self.group)
        sc, rc = cnt.tolist(), rcnt.tolist()
        out = torch.empty((sum(rc), w), dtype=torch.float64, device=dev)
        inp = torch.cat(sends, 0) if sum(sc) else torch.empty((0, w), dtype=torch.float64, device=dev)
        self.dist.all_to_all_single(out.view(-1), inp.reshape(-1), [c * w for c in rc], [c * w for c in sc],
                                    group=self.group)
        return list(torch.split(out, rc, 0))


class ThreadComm(Comm):
    """In-process ranks as threads (tests on one GPU / CPU): exchanges through a shared
    board and a barrier.  Not a stand-in for concurrent GPU kernels: no kernel waits on
    another rank, only the host steps meet at the barrier."""

    class Board:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, board: "ThreadComm.Board", rank: int):
        self.board, self.rank, self.world = board, rank, board.world

    def _exchange(self, item):
        b = self.board
        b.barrier.wait()
        b.slots[self.rank] = item
        b.barrier.wait()
        got = list(b.slots)
        b.barrier.wait()
        return got

    def allreduce(self, t, op):
        got = self._exchange(t)
        out = got[0].clone()
        for g in got[1:]:
            g = g.to(out.device)
            out = out + g if op == "sum" else (torch.minimum(out, g) if op == "min" else torch.maximum(out, g))
        return out

    def alltoallv(self, sends):
        got = self._exchange(sends)
        return [got[s][self.rank].to(sends[0].device) for s in range(self.world)]


def run_threads(world: int, fn):
    """Run fn(comm) for `world` thread-ranks; returns the list of results by rank."""
    board = ThreadComm.Board(world)
    res, err = [None] * world, [None] * world

    def body(r):
        try:
            res[r] = fn(ThreadComm(board, r))
        except BaseException as e:   # surface the failure, release the others
            err[r] = e
            board.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return res


# ---------------------------------------------------------------- backend (product)
class GpuBackend:
    """libdmk on one CUDA device: dmk_plan / dmk_upward / dmk_level_moments / dmk_downward."""

    def __init__(self, device):
        self.device = torch.device(device)

    def plan(self, points, eps, ns, kernel, lam, root, min_level, n_targets=0):
        import paper_2308_00292_b200 as dmk
        return dmk.dmk_plan(points.to(self.device), eps=eps, leaf_capacity=ns, kernel=kernel, lam=lam, root=root,
                            min_level=min_level, n_targets=n_targets)

    def upward(self, plan, charges):
        plan.upward(charges.to(self.device))

    def get_level(self, plan, level):
        p = plan.info().p
        d = torch.empty((8 ** level, p, p, p), dtype=torch.float64, device=self.device)
        return plan.level_moments(level, d)

    def set_level(self, plan, level, dense):
        plan.level_moments(level, dense.to(self.device).contiguous(), set=True)

    def downward(self, plan):
        return plan.downward(device=self.device)

    def close(self, plan):
        plan.close()


# ---------------------------------------------------------------- geometry helpers
def level_codes(x: torch.Tensor, lo: Sequence[float], side: float, level: int) -> torch.Tensor:
    """Morton code of each point's box at `level`, exactly as the library computes keys
    (IEEE subtract, then multiply by 2^21/side, floor, clip; x most significant)."""
    scale = float(2 ** NBITS) / side
    q = torch.floor((x - torch.as_tensor(lo, dtype=torch.float64, device=x.device)) * scale)
    q = torch.clamp(q, 0, 2 ** NBITS - 1).to(torch.int64) >> (NBITS - level)
    code = torch.zeros(x.shape[0], dtype=torch.int64, device=x.device)
    for b in range(level):
        for d in range(3):
            code |= ((q[:, d] >> b) & 1) << (3 * b + (2 - d))
    return code


@functools.lru_cache(maxsize=8)
def colleague_table(level: int) -> np.ndarray:
    """[8^level, 27] Morton codes of the colleagues of every box at `level` (-1 outside)."""
    n1 = 2 ** level
    codes = np.arange(8 ** level, dtype=np.int64)
    c = np.zeros((codes.size, 3), dtype=np.int64)
    for b in range(level):
        for d in range(3):
            c[:, d] |= ((codes >> (3 * b + (2 - d))) & 1) << b
    out = np.full((codes.size, 27), -1, dtype=np.int64)
    k = 0
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                cc = c + np.array([dx, dy, dz])
                ok = np.all((cc >= 0) & (cc < n1), axis=1)
                e = np.zeros(codes.size, dtype=np.int64)
                for b in range(level):
                    for d in range(3):
                        e |= ((cc[:, d] >> b) & 1) << (3 * b + (2 - d))
                out[:, k] = np.where(ok, e, -1)
                k += 1
    return out


def owners_from_histogram(hist: np.ndarray, world: int) -> np.ndarray:
    """Contiguous Morton ranges of boxes with balanced point counts: owner of each box."""
    tot = float(hist.sum())
    if tot == 0:
        return np.zeros(hist.size, dtype=np.int64)
    mid = np.cumsum(hist) - 0.5 * hist
    return np.minimum(world - 1, np.floor(mid * world / tot)).astype(np.int64)


def choose_level(n_total: int, ns: int, world: int) -> int:
    """Partition level Lc: deep enough for ~8 boxes per rank and below the root, at most 4
    (the dense level-(Lc-1) moment exchange is 8^(Lc-1) p^3 doubles)."""
    lv = max(2, math.ceil(math.log(max(8 * world, 2), 8)))
    depth = max(1, math.ceil(math.log(max(n_total / max(ns, 1), 1.0), 8)))
    return int(min(4, max(lv, min(depth, 4))))


# ---------------------------------------------------------------- the distributed evaluation
def dmk_eval_distributed(points: torch.Tensor, charges: torch.Tensor, comm: Comm, backend, eps: float = 1e-6,
                         ns: int = 200, kernel: str = "laplace", lam: float = 0.0, level: int | None = None,
                         stats: dict | None = None) -> torch.Tensor:
    """Potentials at this rank's points (same order), u_i = sum_j K(x_i - x_j) rho_j over
    the points of ALL ranks (coincident pairs omitted).  3D kernels (laplace, yukawa)."""
    dev = points.device
    x = points.to(torch.float64).reshape(-1, 3)
    q = charges.to(torch.float64).reshape(-1)
    n_local = x.shape[0]
    R, me = comm.world, comm.rank
    # 1. root box
    big = torch.tensor([1e300] * 3, dtype=torch.float64, device=dev)
    mn = comm.allreduce(x.min(0).values if n_local else big, "min")
    mx = comm.allreduce(x.max(0).values if n_local else -big, "max")
    lo = mn.tolist()
    ext = float((mx - mn).max())
    side = ext if ext > 0 else 1.0
    n_total = int(comm.allreduce(torch.tensor([float(n_local)], dtype=torch.float64, device=dev), "sum").item())
    Lc = level if level is not None else choose_level(n_total, ns, R)
    if R == 1:   # one rank: the plain single-device evaluation
        plan = backend.plan(x.contiguous(), eps, ns, kernel, lam, None, 0)
        backend.upward(plan, q.contiguous())
        u = torch.as_tensor(backend.downward(plan), device=dev)
        backend.close(plan)
        if stats is not None:
            stats.update(level=0, n_own=n_local, n_halo=0, n_total=n_total)
        return u
    # 2. partition: owners of level-(Lc-1) boxes, inherited by their Lc-children
    code = level_codes(x, lo, side, Lc)
    hist = torch.bincount(code, minlength=8 ** Lc).to(torch.float64)
    hist = comm.allreduce(hist, "sum").cpu().numpy()
    owner_c = owners_from_histogram(hist.reshape(-1, 8).sum(1), R)
    owner = np.repeat(owner_c, 8)
    owner_t = torch.as_tensor(owner, device=dev)
    # 3. exchange to owners: rows [x, y, z, q, src_rank, src_index]
    rows = torch.cat([x, q[:, None], torch.full((n_local, 1), float(me), dtype=torch.float64, device=dev),
                      torch.arange(n_local, dtype=torch.float64, device=dev)[:, None]], 1)
    dst = owner_t[code]
    own = torch.cat(comm.alltoallv([rows[dst == d] for d in range(R)]), 0)
    # 4. halo: owned points to the owners of the colleagues of their Lc-box
    coll = colleague_table(Lc)
    need = np.zeros((8 ** Lc, R), dtype=bool)     # need[c, d]: rank d needs box c as halo
    valid = coll >= 0
    nb_owner = np.where(valid, owner[np.where(valid, coll, 0)], -1)
    for k in range(27):
        ok = nb_owner[:, k] >= 0
        need[np.nonzero(ok)[0], nb_owner[ok, k]] = True
    need[np.arange(8 ** Lc), owner] = False
    need_t = torch.as_tensor(need, device=dev)
    ocode = level_codes(own[:, :3], lo, side, Lc) if own.shape[0] else torch.zeros(0, dtype=torch.int64, device=dev)
    halo = torch.cat(comm.alltoallv([own[need_t[ocode, d]][:, :4] for d in range(R)]), 0)
    n_own, n_halo = own.shape[0], halo.shape[0]
    if stats is not None:
        stats.update(level=Lc, n_own=n_own, n_halo=n_halo, n_total=n_total)
    # 5-7. local evaluation
    p_dense = None
    C = Lc - 1
    if n_own:
        X = torch.cat([own[:, :3], halo[:, :3]], 0).contiguous()
        Q = torch.cat([own[:, 3], halo[:, 3]], 0).contiguous()
        # the halo points are sources only: no local expansions / P2P for their boxes
        plan = backend.plan(X, eps, ns, kernel, lam, lo + [side], Lc, n_own)
        backend.upward(plan, Q)
        p_dense = torch.as_tensor(backend.get_level(plan, C), device=dev)
        mine = torch.as_tensor(owner_c == me, device=dev)
        p_dense = p_dense * mine.reshape((-1,) + (1,) * (p_dense.dim() - 1)).to(p_dense.dtype)
    # ranks without points still take part in the reduction (zeros of the agreed shape)
    shape = torch.tensor(list(p_dense.shape) if p_dense is not None else [0, 0, 0, 0], dtype=torch.float64,
                         device=dev)
    shape = comm.allreduce(shape, "max")
    if p_dense is None:
        p_dense = torch.zeros([int(v) for v in shape.tolist()], dtype=torch.float64, device=dev)
    g_dense = comm.allreduce(torch.as_tensor(p_dense, device=dev), "sum")
    u_own = torch.zeros(0, dtype=torch.float64, device=dev)
    if n_own:
        backend.set_level(plan, C, g_dense)
        u = torch.as_tensor(backend.downward(plan), device=dev)
        u_own = u[:n_own]
        backend.close(plan)
    # 8. return to the source ranks
    srank = own[:, 4].to(torch.int64)
    back = torch.cat([own[:, 5:6], u_own[:, None]], 1)
    got = torch.cat(comm.alltoallv([back[srank == d] for d in range(R)]), 0)
    out = torch.empty(n_local, dtype=torch.float64, device=dev)
    out[got[:, 0].to(torch.int64)] = got[:, 1]
    return out
