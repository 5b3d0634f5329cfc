"""Sharded Strang step (paper_1506_04651_b200/shard.py) on CPU: two gloo ranks
step one BZ problem with the ORACLE as the compute backend (R on cost-balanced Morton intervals, D on
species i mod P, A replicated), and must reproduce the single-process oracle step bit for bit — the
per-leaf reaction and the per-species diffusion do not depend on the partition.  Also pins the
partition rule of include/rdmr.h (rd_shard_bounds) in plain numpy."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def ref_bounds(cost, p):
    """include/rdmr.h rd_shard_bounds, written out: w = max(cost, 0) + 1, S_i = sum_{c<i} w_c,
    bounds[k] = min{i : p S_i >= k W} (exact integers)."""
    n = len(cost)
    w = (np.maximum(np.asarray(cost, dtype=np.int64), 0) + 1) if cost is not None else np.ones(n, dtype=np.int64)
    S = np.concatenate([[0], np.cumsum(w)])
    W = int(S[-1])
    out = [0]
    for k in range(1, p):
        out.append(int(np.searchsorted(p * S, k * W, side="left")))
    out.append(n)
    return out


def test_ref_bounds_properties():
    rng = np.random.default_rng(7)
    for n, p in [(0, 3), (1, 4), (5, 8), (1000, 2), (1000, 7), (4097, 8)]:
        cost = rng.integers(0, 65536, n)
        b = ref_bounds(cost, p)
        assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
        if n:
            w = cost + 1
            W, wmax = w.sum(), w.max()
            for k in range(p):
                part = w[b[k]:b[k + 1]].sum()
                assert abs(part - W / p) <= wmax
    assert ref_bounds([0] * 10, 4) == [0, 3, 5, 8, 10]  # equal weights: ceil(k n / p)
    assert ref_bounds([-5, 0, 0, 0], 2) == [0, 2, 4]  # negative costs count as 0


class OracleBackend:
    """The oracle as the shard compute backend (test infrastructure only)."""

    def __init__(self, orc, o, model, nthreads=4):
        self.orc, self.o, self.model, self.nt = orc, o, model, nthreads

    def values(self):
        return torch.from_numpy(self.o.leaves()[1].copy())

    def commit(self, u):
        self.o.set_values(u.numpy())

    def bounds(self, u, p):
        cost = (np.abs(u[0].numpy()) * 4096).astype(np.int64)  # any deterministic cost exercises balancing
        return ref_bounds(cost, p)

    def react(self, u_part, T):
        y, _, st = self.orc.radau5(u_part.numpy(), self.model, T, nthreads=self.nt)
        assert (st == 0).all()
        u_part.copy_(torch.from_numpy(y))

    def diffuse(self, eps, T):
        self.o.diffuse(eps, T, nthreads=self.nt)

    def adapt(self):
        self.o.adapt()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(orc):
    import synth
    w = synth.cfg3(J=6, K=3)
    o = orc.Grid.build(2, w.level_min, w.level_max, w.eps_mr, w.u.reshape(w.m, -1))
    return w, o, orc.Model(dict(w.model, m=w.m))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import oracle as orc
    from paper_1506_04651_b200.shard import ShardedStrang
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, o, M = _problem(orc)
        S = ShardedStrang(OracleBackend(orc, o, M), w.eps_diff)
        res = []
        for scheme in (0, 1):
            S.step(w.dt, scheme)
            k, u = o.leaves()
            res.append((k.copy(), u.copy(), list(S.last_bounds)))
            S.adapt()
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_strang_matches_single_process(orc, world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    w, o, M = _problem(orc)
    for it, scheme in enumerate((0, 1)):
        assert o.strang(M, w.eps_diff, w.dt, scheme, nthreads=4) == 0
        k, u = o.leaves()
        for r in range(world):
            rk, ru, bnd = out[r][it]
            assert np.array_equal(rk, k)
            assert np.array_equal(ru, u), (r, it, np.abs(ru - u).max())
            assert len(bnd) == world + 1 and bnd[0] == 0 and bnd[-1] == len(k)
            assert all(bnd[i] < bnd[i + 1] for i in range(world))  # every rank had work
        o.adapt()
