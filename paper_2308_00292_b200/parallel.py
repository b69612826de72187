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

    def get_boxes(self, plan, level, codes):
        p = plan.info().p
        codes = torch.as_tensor(codes, dtype=torch.int64, device=self.device)
        out = torch.empty((codes.numel(), p, p, p), dtype=torch.float64, device=self.device)
        return plan.box_moments(level, codes, out)

    def set_boxes(self, plan, level, codes, values):
        codes = torch.as_tensor(codes, dtype=torch.int64, device=self.device)
        plan.box_moments(level, codes, values.to(self.device).contiguous(), set=True)

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


# ---------------------------------------------------------------- locally essential tree
def morton_encode(ix: torch.Tensor, iy: torch.Tensor, iz: torch.Tensor, level: int) -> torch.Tensor:
    code = torch.zeros_like(ix)
    for b in range(level):
        code |= (((ix >> b) & 1) << (3 * b + 2)) | (((iy >> b) & 1) << (3 * b + 1)) | (((iz >> b) & 1) << (3 * b))
    return code


def morton_decode(code: torch.Tensor, level: int):
    ix, iy, iz = torch.zeros_like(code), torch.zeros_like(code), torch.zeros_like(code)
    for b in range(level):
        ix |= ((code >> (3 * b + 2)) & 1) << b
        iy |= ((code >> (3 * b + 1)) & 1) << b
        iz |= ((code >> (3 * b)) & 1) << b
    return ix, iy, iz


def neighbour_codes(code: torch.Tensor, level: int) -> torch.Tensor:
    """[n, 27] Morton codes of the colleagues (incl. itself) of boxes `code` at `level`,
    -1 outside the root box; slot (dx+1)*9 + (dy+1)*3 + (dz+1)."""
    ix, iy, iz = morton_decode(code, level)
    n1 = 1 << level
    out = []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                jx, jy, jz = ix + dx, iy + dy, iz + dz
                ok = (jx >= 0) & (jx < n1) & (jy >= 0) & (jy < n1) & (jz >= 0) & (jz < n1)
                c = morton_encode(jx.clamp(0, n1 - 1), jy.clamp(0, n1 - 1), jz.clamp(0, n1 - 1), level)
                out.append(torch.where(ok, c, torch.full_like(c, -1)))
    return torch.stack(out, 1)


def choose_let_levels(n_total: int, ns: int, world: int) -> int:
    """Halo level Lh = the plans' min_level <= 6: the particle halo is one level-Lh box
    thick; as deep as the tree allows (one level above the leaves of a uniform cloud)."""
    depth = max(1, math.ceil(math.log(max(n_total / max(ns, 1), 1.0), 8)))
    return int(min(6, max(2, depth - 1)))


KEY_BITS = 3 * NBITS   # 63-bit Morton keys, as the library sorts


def box_rank_bits(code: torch.Tensor, level: int, splitters: torch.Tensor) -> torch.Tensor:
    """Bitmask of the ranks whose Morton-key range meets box `code` of `level` (rank r
    owns the keys in [splitters[r-1], splitters[r]))."""
    span = 3 * (NBITS - level)
    k0, k1 = code << span, ((code + 1) << span) - 1
    r0 = torch.searchsorted(splitters, k0, right=True)
    r1 = torch.searchsorted(splitters, k1, right=True)
    one = torch.ones_like(code)
    return ((one << (r1 + 1)) - 1) ^ ((one << r0) - 1)


def key_splitters(keys: torch.Tensor, comm: Comm, samples: int = 256) -> torch.Tensor:
    """R - 1 Morton-key splitters of all ranks' points by sample sort: every rank
    contributes `samples` evenly spaced keys of its sorted keys; the merged sample's
    R-quantiles split the points into R contiguous ranges of ~N/R points."""
    R = comm.world
    dev = keys.device
    n = keys.shape[0]
    ks = torch.sort(keys).values
    cnt = comm.allreduce(torch.tensor([float(n)], dtype=torch.float64, device=dev), "sum")
    # weights: each sample stands for n/samples local points
    if n:
        idx = torch.clamp(((torch.arange(samples, device=dev) + 0.5) * n / samples).to(torch.int64), max=n - 1)
        smp = (ks[idx] >> 10).to(torch.float64)   # 53-bit: exact in float64
        w = torch.full((samples,), n / samples, dtype=torch.float64, device=dev)
    else:
        smp = torch.zeros(samples, dtype=torch.float64, device=dev)
        w = torch.zeros(samples, dtype=torch.float64, device=dev)
    # gather every rank's (sample, weight) through the all-reduce of a rank-indexed table
    tab = torch.zeros((R, 2, samples), dtype=torch.float64, device=dev)
    tab[comm.rank, 0] = smp
    tab[comm.rank, 1] = w
    tab = comm.allreduce(tab, "sum")
    allk, allw = tab[:, 0].reshape(-1), tab[:, 1].reshape(-1)
    order = torch.argsort(allk)
    allk, cw = allk[order], torch.cumsum(allw[order], 0)
    tot = float(cnt.item())
    pos = torch.searchsorted(cw, torch.arange(1, R, device=dev, dtype=torch.float64) * tot / R)
    return allk[pos.clamp(max=allk.shape[0] - 1)].to(torch.int64) << 10


def let_halo_fraction(hist_h: np.ndarray, Lh: int, world: int) -> np.ndarray:
    """Halo points / owned points per rank for the point counts of every level-Lh box,
    with the partition and halo rules of dmk_eval_let (no points needed): ranks own
    contiguous Morton ranges of N/R points; a rank receives, as halo, the other ranks'
    points in every level-Lh box equal or adjacent to a box holding its points."""
    h = torch.as_tensor(hist_h, dtype=torch.float64)
    cs = torch.cumsum(h, 0)
    tot = float(cs[-1])
    b0, b1 = cs - h, cs
    code = torch.arange(8 ** Lh, dtype=torch.int64)
    nb = neighbour_codes(code, Lh)
    frac = np.zeros(world)
    for r in range(world):
        a, b = r * tot / world, (r + 1) * tot / world
        mine = torch.clamp(torch.minimum(b1, torch.full_like(b1, b)) - torch.maximum(b0, torch.full_like(b0, a)), min=0)
        has = mine > 0
        need = torch.zeros(8 ** Lh, dtype=torch.bool)
        for k in range(27):
            ok = nb[:, k] >= 0
            need[nb[ok, k][has[ok]]] = True
        frac[r] = float((h[need] - mine[need]).sum()) / max(float(mine.sum()), 1.0)
    return frac


def dmk_eval_let(points: torch.Tensor, charges: torch.Tensor, comm: Comm, backend, eps: float = 1e-6,
                 ns: int = 200, kernel: str = "laplace", lam: float = 0.0, levels=None,
                 stats: dict | None = None) -> torch.Tensor:
    """The distributed evaluation with a locally essential tree (north star's data plane):
    potentials at this rank's points (same order) over the points of ALL ranks.

      1. root box: all-reduce of the bounds (reading R5's single-process root cube).
      2. ownership: contiguous Morton-key ranges of ~N/R points (sample-sort splitters,
         all-reduced sample); every point goes to its owner (all-to-all).  Boxes on a
         range boundary are shared.
      3. particle halo, one level-Lh box thick: an owned point also goes to every rank with
         points in its level-Lh box or in one of that box's colleagues (all-to-all) -- the
         neighbour-halo particles: every level-Lh box holding owned points, its colleagues,
         and so every colleague (level >= Lh) and direct-list source of an owned leaf (all
         leaves are at level >= Lh, the plan's forced levels) are whole locally.
      4. local plan over own + halo points, shared root, min_level = Lh, targets = own.
      5. upward with the halo charges zeroed: exact owned-only (partial) moments.  Dense
         level Gd = min(3, Lh - 1): all-reduce SUM (the replicated coarse levels).  Levels
         Gd+1..Lh-1: the partial moments of each box holding owned points go to every rank
         with points in one of its colleagues (all-to-all), which sums them -- the
         boundary proxy data (sparse, one layer of boxes per level).
      6. upward with all charges, then set the received boundary moments and the reduced
         dense level (which rebuilds the levels above it by T_c2p), downward, and return
         the own potentials to the ranks the points came from (all-to-all).
    """
    dev = points.device
    x = points.to(torch.float64).reshape(-1, 3)
    q = charges.to(torch.float64).reshape(-1)
    n_local = x.shape[0]
    R, me = comm.world, comm.rank
    big = torch.tensor([1e300] * 3, dtype=torch.float64, device=dev)
    mn = comm.allreduce(x.min(0).values if n_local else big, "min")
    mx = comm.allreduce(x.max(0).values if n_local else -big, "max")
    lo = mn.tolist()
    ext = float((mx - mn).max())
    side = ext if ext > 0 else 1.0
    n_total = int(comm.allreduce(torch.tensor([float(n_local)], dtype=torch.float64, device=dev), "sum").item())
    Lh = int(levels) if levels is not None else choose_let_levels(n_total, ns, R)
    if not (1 <= Lh <= 6):
        raise ValueError(f"LET halo level must be in [1, 6], got {Lh}")
    if R == 1:
        plan = backend.plan(x.contiguous(), eps, ns, kernel, lam, None, 0)
        backend.upward(plan, q.contiguous())
        u = torch.as_tensor(backend.downward(plan), device=dev)
        backend.close(plan)
        if stats is not None:
            stats.update(level=0, n_own=n_local, n_halo=0, n_total=n_total)
        return u
    Gd = min(3, Lh - 1)   # dense all-reduce level
    sh = 3 * (NBITS - Lh)
    # 2. ownership: contiguous Morton-key ranges of ~N/R points (sample-sort splitters)
    key = level_codes(x, lo, side, NBITS)
    splitters = key_splitters(key, comm)
    rows = torch.cat([x, q[:, None], torch.full((n_local, 1), float(me), dtype=torch.float64, device=dev),
                      torch.arange(n_local, dtype=torch.float64, device=dev)[:, None]], 1)
    dst = torch.searchsorted(splitters, key, right=True)
    own = torch.cat(comm.alltoallv([rows[dst == d] for d in range(R)]), 0)
    n_own = own.shape[0]
    # 3. halo: every rank with points in a level-Lh colleague (or the box itself) of an
    # owned point's box gets the point
    ocode = (level_codes(own[:, :3], lo, side, NBITS) >> sh) if n_own else torch.zeros(0, dtype=torch.int64,
                                                                                            device=dev)
    ubox, inv = torch.unique(ocode, return_inverse=True)
    nb = neighbour_codes(ubox, Lh)                                   # [nbox, 27]
    dest = torch.zeros(len(ubox), dtype=torch.int64, device=dev)
    for k in range(27):
        bk = box_rank_bits(nb[:, k].clamp(min=0), Lh, splitters)
        dest |= torch.where(nb[:, k] >= 0, bk, torch.zeros_like(bk))
    sends = []
    for d in range(R):
        if d == me or n_own == 0:
            sends.append(own[:0, :4])
            continue
        sends.append(own[((dest >> d) & 1).bool()[inv]][:, :4])
    halo = torch.cat(comm.alltoallv(sends), 0)
    n_halo = halo.shape[0]
    if stats is not None:
        stats.update(level=Lh, n_own=n_own, n_halo=n_halo, n_total=n_total)
    # 4.-5. local plan, owned-only upward, dense + boundary exchanges
    X = torch.cat([own[:, :3], halo[:, :3]], 0).contiguous()
    Qall = torch.cat([own[:, 3], halo[:, 3]], 0).contiguous()
    Qown = torch.cat([own[:, 3], torch.zeros(n_halo, dtype=torch.float64, device=dev)], 0).contiguous()
    plan = backend.plan(X, eps, ns, kernel, lam, lo + [side], Lh, n_own) if n_own else None
    if plan is not None:
        backend.upward(plan, Qown)
        dense = torch.as_tensor(backend.get_level(plan, Gd), device=dev)
    else:
        dense = None
    shape = torch.tensor(list(dense.shape) if dense is not None else [0, 0, 0, 0], dtype=torch.float64, device=dev)
    shape = comm.allreduce(shape, "max")
    p = int(shape[1].item())
    p3 = p ** 3
    if dense is None:
        dense = torch.zeros([int(v) for v in shape.tolist()], dtype=torch.float64, device=dev)
    g_dense = comm.allreduce(dense, "sum")
    # boundary exchange, levels Gd+1 .. Lh-1: the owned-only (partial) moments of every box
    # holding owned points go to every rank with points in one of the box's colleagues;
    # each rank sums what it receives with its own partial -> complete moments of every
    # box it needs (colleagues of the ancestors of its points)
    complete = {}
    for lv in range(Gd + 1, Lh):
        mine = torch.unique(ocode >> (3 * (Lh - lv))) if n_own else torch.zeros(0, dtype=torch.int64, device=dev)
        vals = (torch.as_tensor(backend.get_boxes(plan, lv, mine), device=dev).reshape(-1, p3)
                if len(mine) else torch.zeros((0, p3), dtype=torch.float64, device=dev))
        nbl = neighbour_codes(mine, lv)
        dest = torch.zeros(len(mine), dtype=torch.int64, device=dev)
        for k in range(27):
            bk = box_rank_bits(nbl[:, k].clamp(min=0), lv, splitters)
            dest |= torch.where(nbl[:, k] >= 0, bk, torch.zeros_like(bk))
        sends = []
        for d in range(R):
            m = ((dest >> d) & 1).bool() if d != me else torch.zeros(len(mine), dtype=torch.bool, device=dev)
            sends.append(torch.cat([mine[m].to(torch.float64)[:, None], vals[m]], 1))
        got = torch.cat(comm.alltoallv(sends), 0)
        need = torch.unique(nbl[nbl >= 0]) if len(mine) else torch.zeros(0, dtype=torch.int64, device=dev)
        acc = torch.zeros((len(need), p3), dtype=torch.float64, device=dev)
        if len(need):
            pos = torch.searchsorted(need, mine)
            acc.index_add_(0, pos, vals)
            gc = got[:, 0].to(torch.int64)
            pos = torch.searchsorted(need, gc)
            ok = (pos < len(need)) & (need[pos.clamp(max=len(need) - 1)] == gc)
            acc.index_add_(0, pos[ok], got[ok, 1:])
        complete[lv] = (need, acc)
    u_own = torch.zeros(0, dtype=torch.float64, device=dev)
    if plan is not None:
        backend.upward(plan, Qall)
        for lv in range(Gd + 1, Lh):
            need, acc = complete[lv]
            if len(need):
                backend.set_boxes(plan, lv, need, acc.reshape(-1, p, p, p))
        backend.set_level(plan, Gd, g_dense)
        u = torch.as_tensor(backend.downward(plan), device=dev)
        u_own = u[:n_own]
        backend.close(plan)
    # 6. return to the source ranks
    srank = own[:, 4].to(torch.int64)
    back = torch.cat([own[:, 5:6], u_own[:, None]], 1)
    got = torch.cat(comm.alltoallv([back[srank == d] for d in range(R)]), 0)
    out = torch.empty(n_local, dtype=torch.float64, device=dev)
    out[got[:, 0].to(torch.int64)] = got[:, 1]
    return out
