"""The distributed DMK driver (paper_2308_00292_b200/parallel.py) on CPU: partition
helpers against brute force, and the whole N > 1 path -- root all-reduce, Morton
partition, all-to-all exchange, halo, coarse-moment all-reduce, return exchange -- with
torch.distributed gloo at world size 2 (and thread ranks at world size 3), the per-rank
compute done by the oracle (tests/oracle_backend.py)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

import dmk_inputs
from oracle import direct
from oracle.dmk import dmk
from oracle.tree import Tree
from paper_2308_00292_b200 import parallel as par

from oracle_backend import OracleBackend

EPS, NS = 1e-6, 30


def test_level_codes_match_oracle_tree_keys():
    x, _ = dmk_inputs.clusters(3000, seed=2)
    T = Tree(x, 50)
    for L in (1, 2, 3):
        got = par.level_codes(torch.as_tensor(x), T.lo.tolist(), T.side, L).numpy()
        ref = np.empty(len(x), dtype=np.int64)
        ref[T.perm] = T.keys >> (3 * (21 - L))
        assert np.array_equal(got, ref)


def test_colleague_table_brute_force():
    L = 2
    tab = par.colleague_table(L)
    from oracle.tree import decode, encode
    for c in range(8 ** L):
        xc = decode(np.array([c]), L)[0]
        want = set()
        for off in np.ndindex(3, 3, 3):
            cc = xc + np.array(off) - 1
            if np.all((cc >= 0) & (cc < 2 ** L)):
                want.add(int(encode(cc, L)[0]))
        assert set(int(v) for v in tab[c] if v >= 0) == want


def test_owners_balanced_and_contiguous():
    rng = np.random.default_rng(0)
    h = rng.integers(0, 100, 512).astype(float)
    for R in (1, 2, 3, 8):
        o = par.owners_from_histogram(h, R)
        assert np.all(np.diff(o) >= 0) and o.min() == 0 and o.max() <= R - 1
        loads = np.bincount(o, weights=h, minlength=R)
        assert np.max(loads) <= h.sum() / R + h.max() + 1e-9


def split(n, world, seed):
    """An arbitrary (non-Morton) split of the points over the ranks."""
    return np.random.default_rng(seed).integers(0, world, n)


def reference(x, q, L):
    """Single-process oracle DMK with the root and min_level the ranks share."""
    lo = x.min(0)
    side = float((x.max(0) - lo).max())
    return dmk(x, q, EPS, NS, "laplace", 0.0, root=list(lo) + [side], min_level=L)


def test_thread_ranks_world3_oracle():
    x, q = dmk_inputs.clusters(2500, seed=4)
    who = split(len(x), 3, 1)

    def fn(comm):
        m = who == comm.rank
        st = {}
        u = par.dmk_eval_distributed(torch.as_tensor(x[m]), torch.as_tensor(q[m]), comm, OracleBackend(), eps=EPS,
                                     ns=NS, level=2, stats=st)
        return u.numpy(), st

    res = par.run_threads(3, fn)
    u = np.empty(len(x))
    for r in range(3):
        u[who == r] = res[r][0]
    assert sum(r[1]["n_own"] for r in res) == len(x)
    assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2 * EPS
    assert direct.rel_l2(u, reference(x, q, 2)) <= EPS


def _gloo_worker(rank, world, port, path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, q = dmk_inputs.uniform(3000, seed=6)
    who = split(len(x), world, 2)
    m = who == rank
    st = {}
    u = par.dmk_eval_distributed(torch.as_tensor(x[m]), torch.as_tensor(q[m]), par.TorchComm(), OracleBackend(),
                                 eps=EPS, ns=NS, level=2, stats=st)
    np.save(os.path.join(path, f"u{rank}.npy"), u.numpy())
    np.save(os.path.join(path, f"s{rank}.npy"), np.array([st["n_own"], st["n_halo"]]))
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_oracle():
    """world_size 2 over torch.distributed gloo (the NCCL path's host logic on CPU)."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, free_port(), d), nprocs=2, join=True)
        x, q = dmk_inputs.uniform(3000, seed=6)
        who = split(len(x), 2, 2)
        u = np.empty(len(x))
        for r in range(2):
            u[who == r] = np.load(os.path.join(d, f"u{r}.npy"))
        st = [np.load(os.path.join(d, f"s{r}.npy")) for r in range(2)]
    assert st[0][0] + st[1][0] == len(x) and st[0][0] > 0 and st[1][0] > 0
    assert st[0][1] > 0 and st[1][1] > 0          # both ranks received halo particles
    assert direct.rel_l2(u, direct.laplace3d(x, q)) <= 2 * EPS
    assert direct.rel_l2(u, reference(x, q, 2)) <= EPS
