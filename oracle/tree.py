"""Level-restricted adaptive 2^d-tree (d = 3 octree, d = 2 quadtree) and interaction
lists  (oracle; test infrastructure).

Paper: Sec. 3.2 (adaptive refinement until a leaf holds at most
n_s points, level restriction, colleagues C(B), coarse neighbours N(B)),
Sec. 3.3 (fine neighbours F(B); the residual kernel index is
the SOURCE box level), Fig. 7 caption (list L_D of a leaf S
at level l = all target boxes that are its neighbours at level l or leaf
neighbours at level l-1) and Sec. 3.5 Step 0 / flags.

Conventions (readings R5-R8 in DESIGN.md):
  * Root cube: lo_d = min_i x_{i,d}; side = max_d (max_i x_{i,d} - lo_d) (1 if 0).
    Integer coordinates q_d = floor((x_d - lo_d) * (2^21 / side)) clipped to
    [0, 2^21 - 1]; Morton key interleaves bits with x most significant in each
    d-tuple (63-bit keys in 3D, 42-bit in 2D).  Points are stably sorted by key.
  * Everything below holds for d = 2 with 4 children / 9 colleagues in place of
    8 / 27 (the paper's algorithm is stated for general d, Sec. 3.5).
  * A box is refined iff it holds more than n_s points (sources = targets) and its
    level is < LMAX.  "Share a boundary point" = closed boxes intersect.
  * 2:1 balance (level restriction): any level-l box that touches a non-leaf box
    of level l+1 is itself non-leaf.  Fixpoint built bottom-up.
  * Boxes kept: all non-leaf boxes (even if empty) and all non-empty leaves.
  * F_out(B) = non-leaf and non-empty (reading R6; the paper's "> n_s sources"
    flag, extended to balance-split boxes so that every D_l term has an owner).
  * Plane-wave list of a non-empty box B at level l: F_out colleagues of B.
  * Direct (residual) list of a non-empty leaf B at level L (gather form of the
    paper's L_D): non-empty leaves S at level l <= L that are colleagues of
    B's level-l ancestor, plus non-empty leaves at level L+1 touching B.
"""
from __future__ import annotations

import itertools

import numpy as np

NBITS = 21          # bits per coordinate in the 63-bit Morton key
LMAX = 20           # deepest level a box may be refined into


def normalize(points: np.ndarray, root=None):
    """Root cube and integer coordinates (reading R5).  Returns (lo, side, q).
    root = (lo_0, .., lo_{d-1}, side) fixes the cube (a distributed evaluation)."""
    x = np.asarray(points, dtype=np.float64)
    if root is not None:
        d = x.shape[1]
        lo, side = np.asarray(root[:d], dtype=np.float64), float(root[d])
    else:
        lo = x.min(axis=0)
        ext = (x.max(axis=0) - lo).max()
        side = float(ext) if ext > 0 else 1.0
    scale = float(2 ** NBITS) / side
    q = np.floor((x - lo) * scale)
    q = np.clip(q, 0, 2 ** NBITS - 1).astype(np.int64)
    return lo, side, q


def morton(q: np.ndarray) -> np.ndarray:
    """Morton key of integer coordinates q (n, d); bit d b + (d-1-k) = coordinate k bit b."""
    n, d = q.shape
    key = np.zeros(n, dtype=np.int64)
    for b in range(NBITS):
        for k in range(d):
            key |= ((q[:, k] >> b) & 1) << (d * b + (d - 1 - k))
    return key


def decode(code: np.ndarray, level: int, d: int = 3) -> np.ndarray:
    """Box code at `level` -> integer box coordinates (n, d)."""
    code = np.asarray(code, dtype=np.int64)
    out = np.zeros((code.shape[0], d), dtype=np.int64)
    for b in range(level):
        for k in range(d):
            out[:, k] |= ((code >> (d * b + (d - 1 - k))) & 1) << b
    return out


def encode(c: np.ndarray, level: int, d: int = 3) -> np.ndarray:
    c = np.asarray(c, dtype=np.int64).reshape(-1, d)
    code = np.zeros(c.shape[0], dtype=np.int64)
    for b in range(level):
        for k in range(d):
            code |= ((c[:, k] >> b) & 1) << (d * b + (d - 1 - k))
    return code


def morton3(q):
    return morton(q)


def decode3(code, level):
    return decode(code, level, 3)


def encode3(c, level):
    return encode(c, level, 3)


class Tree:
    """Adaptive, level-restricted 2^d-tree over one point set (sources = targets)."""

    def __init__(self, points: np.ndarray, ns: int, root=None, min_level: int = 0):
        """root: fixed root cube (lo..., side); min_level: every box of levels < min_level
        exists and is refined, empty or not (the shared coarse tree of a distributed
        evaluation, paper_2308_00292_b200/parallel.py)."""
        pts = np.asarray(points, dtype=np.float64)
        self.N, self.d = pts.shape
        self.nch, self.ncol = 2 ** self.d, 3 ** self.d
        self.ns = int(ns)
        self.min_level = int(min_level)
        self.lo, self.side, q = normalize(pts, root)
        key = morton(q)
        self.perm = np.argsort(key, kind="stable")          # sorted -> original
        self.keys = key[self.perm]
        self.xs = (pts[self.perm] - self.lo) / self.side     # normalised coords in [0,1]^d
        self._build()

    # ------------------------------------------------------------------
    def _codes(self, l):
        return self.keys >> (self.d * (NBITS - l))

    def _build(self):
        N, ns = self.N, self.ns
        # unbalanced refinement: U[l] = level-l boxes holding > ns points
        U = []
        for l in range(0, LMAX):
            if l < self.min_level:
                U.append(np.arange(2 ** (self.d * l), dtype=np.int64))
                continue
            if N == 0:
                break
            uq, cnt = np.unique(self._codes(l), return_counts=True)
            sel = uq[cnt > ns]
            if sel.size == 0:
                break
            U.append(sel)
        ltop = len(U) - 1
        # 2:1 balance, bottom-up: B[l] = U[l] + level-l boxes touching B[l+1]
        B = [None] * (ltop + 1)
        if ltop >= 0:
            B[ltop] = U[ltop]
            for l in range(ltop - 1, -1, -1):
                qc = decode(B[l + 1], l + 1, self.d)
                lo_ = np.where(qc % 2 == 0, qc // 2 - 1, qc // 2)    # touching range per dim
                cands = [U[l]]
                n1 = 2 ** l
                for o in itertools.product(range(2), repeat=self.d):
                    cc = lo_ + np.array(o)
                    ok = np.all((cc >= 0) & (cc < n1), axis=1)
                    cands.append(encode(cc[ok], l, self.d))
                B[l] = np.unique(np.concatenate(cands))
        self.nonleaf = B
        self.nlevels = ltop + 2 if ltop >= 0 else 1           # levels 0..nlevels-1 hold boxes
        # box sets per level
        levels, codes = [], []
        for l in range(self.nlevels):
            if l == 0:
                cl = np.array([0], dtype=np.int64)
            else:
                par = self._codes(l - 1)
                nonempty = np.unique(self._codes(l)[np.isin(par, B[l - 1])])
                extra = B[l] if l <= ltop else np.zeros(0, dtype=np.int64)
                cl = np.unique(np.concatenate([nonempty, extra]))
            levels.append(np.full(cl.shape, l, dtype=np.int64))
            codes.append(cl)
        self.level_offset = np.concatenate([[0], np.cumsum([len(c) for c in codes])])
        self.box_level = np.concatenate(levels)
        self.box_code = np.concatenate(codes)
        nb = self.nbox = self.box_code.shape[0]
        self.box_coords = np.zeros((nb, self.d), dtype=np.int64)
        self.box_leaf = np.zeros(nb, dtype=bool)
        self.box_start = np.zeros(nb, dtype=np.int64)
        self.box_end = np.zeros(nb, dtype=np.int64)
        for l in range(self.nlevels):
            a, b = self.level_offset[l], self.level_offset[l + 1]
            cl = self.box_code[a:b]
            self.box_coords[a:b] = decode(cl, l, self.d)
            self.box_leaf[a:b] = ~np.isin(cl, B[l]) if l <= ltop else True
            codes_l = self._codes(l)
            self.box_start[a:b] = np.searchsorted(codes_l, cl, side="left")
            self.box_end[a:b] = np.searchsorted(codes_l, cl, side="right")
        self.box_npts = self.box_end - self.box_start
        # parent / children / colleagues
        self.box_parent = np.full(nb, -1, dtype=np.int64)
        self.box_children = np.full((nb, self.nch), -1, dtype=np.int64)
        self.box_colleagues = np.full((nb, self.ncol), -1, dtype=np.int64)
        for i in range(nb):
            l = self.box_level[i]
            if l > 0:
                p = self.find(l - 1, self.box_code[i] >> self.d)
                self.box_parent[i] = p
                self.box_children[p, self.box_code[i] & (self.nch - 1)] = i
        for i in range(nb):
            l = self.box_level[i]
            c = self.box_coords[i]
            # colleague slot k enumerates offsets in {-1,0,1}^d, last axis fastest
            for k, off in enumerate(itertools.product((-1, 0, 1), repeat=self.d)):
                cc = c + np.array(off)
                if np.all((cc >= 0) & (cc < 2 ** l)):
                    self.box_colleagues[i, k] = self.find(l, encode(cc, l, self.d)[0])
        # F_out: non-leaf and non-empty (reading R6), or forced (level < min_level)
        self.fout = (~self.box_leaf) & ((self.box_npts > 0) | (self.box_level < self.min_level))
        # leaf of every (sorted) point
        self.point_leaf = np.full(self.N, -1, dtype=np.int64)
        for i in np.nonzero(self.box_leaf)[0]:
            self.point_leaf[self.box_start[i]:self.box_end[i]] = i
        self._lists()

    def find(self, l: int, code: int) -> int:
        """Index of the box with `code` at level l, or -1."""
        a, b = self.level_offset[l], self.level_offset[l + 1]
        j = np.searchsorted(self.box_code[a:b], code)
        if j < b - a and self.box_code[a + j] == code:
            return int(a + j)
        return -1

    def center(self, i: int) -> np.ndarray:
        s = 2.0 ** (-int(self.box_level[i]))
        return (self.box_coords[i] + 0.5) * s

    def ancestor(self, i: int, l: int) -> int:
        while self.box_level[i] > l:
            i = self.box_parent[i]
        return int(i)

    def _lists(self):
        nb = self.nbox
        self.pwlist = [[] for _ in range(nb)]
        self.dlist = [[] for _ in range(nb)]
        for i in range(nb):
            if self.box_npts[i] == 0:
                continue
            self.pwlist[i] = [int(s) for s in self.box_colleagues[i] if s >= 0 and self.fout[s]]
        self.fin = np.array([len(self.pwlist[i]) > 0 for i in range(nb)])
        for i in range(nb):
            if not self.box_leaf[i] or self.box_npts[i] == 0:
                continue
            L = int(self.box_level[i])
            lst = set()
            for l in range(L, -1, -1):
                a = self.ancestor(i, l)
                for s in self.box_colleagues[a]:
                    if s >= 0 and self.box_leaf[s] and self.box_npts[s] > 0:
                        lst.add(int(s))
            # fine neighbours: leaves at level L+1 touching B
            c = self.box_coords[i]
            for s in self.box_colleagues[i]:
                if s < 0 or self.box_leaf[s]:
                    continue
                for ch in self.box_children[s]:
                    if ch < 0 or not self.box_leaf[ch] or self.box_npts[ch] == 0:
                        continue
                    cc = self.box_coords[ch]
                    if np.all((cc >= 2 * c - 1) & (cc <= 2 * c + 2)):
                        lst.add(int(ch))
            self.dlist[i] = sorted(lst)
