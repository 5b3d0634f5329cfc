"""GPU parity of the sharded-Strang building blocks through the C ABI:
rd_shard_bounds against its integer definition, rd_reaction_radau5_cells on intervals / cell lists against
the whole-field call (bit for bit: the per-cell arithmetic does not depend on the partition), the
species split of D, and a ShardedStrang step on one rank against rd_strang_step."""
import numpy as np
import pytest

import synth
from tests.test_gpu_mr_rock4 import gpu_build, gpu_leaves
from tests.test_shard import ref_bounds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def test_shard_bounds_vs_definition(P):
    import torch
    rng = np.random.default_rng(3)
    for n in (0, 1, 5, 1000, 200001):
        cost = rng.integers(0, 65536, n).astype(np.int32)
        cost[: n // 7] = 0
        ct = torch.tensor(cost, device="cuda")
        for p in (1, 2, 3, 8, 148):
            assert P.rd_shard_bounds(n, ct, p) == ref_bounds(cost, p), (n, p)
            assert P.rd_shard_bounds(n, None, p) == ref_bounds(np.zeros(n, dtype=np.int64), p)
    with pytest.raises(P.RdError):
        P.rd_shard_bounds(10, None, 0)


def _bz_field(n, seed):
    return synth.random_bz_cells(n, seed)


def test_reaction_cells_interval_and_order(P):
    import torch
    u0 = _bz_field(20000, 71)
    M = P.Model(dict(kind="oregonator", **synth.OREGONATOR))
    full = torch.tensor(u0, device="cuda")
    P.rd_reaction_radau5(full, M, 1e-3)
    full = full.cpu().numpy()
    # interval [a, b) of the [3, N] field
    a, b = 1234, 15678
    u = torch.tensor(u0, device="cuda")
    cnt = torch.zeros((8, u.shape[1]), dtype=torch.int32, device="cuda")
    P.rd_reaction_radau5_cells(u[:, a:b], M, 1e-3, cell_counters=cnt[:, a:b])
    got = u.cpu().numpy()
    assert np.array_equal(got[:, a:b], full[:, a:b])
    assert np.array_equal(got[:, :a], u0[:, :a]) and np.array_equal(got[:, b:], u0[:, b:])
    c = cnt.cpu().numpy()
    assert (c[0, a:b] > 0).all() and not c[:, :a].any() and not c[:, b:].any()
    # a scattered cell list, in a scrambled order
    sel = np.random.default_rng(4).choice(u0.shape[1], 777, replace=False).astype(np.int32)
    u = torch.tensor(u0, device="cuda")
    P.rd_reaction_radau5_cells(u, M, 1e-3, order=torch.tensor(sel, device="cuda"))
    got = u.cpu().numpy()
    mask = np.zeros(u0.shape[1], dtype=bool)
    mask[sel] = True
    assert np.array_equal(got[:, mask], full[:, mask]) and np.array_equal(got[:, ~mask], u0[:, ~mask])


def test_reaction_cells_warp_kernel(P):
    """The warp-per-cell kernel (m = 20, BJ configs[4] network) on an interval and on a cell list of a
    [20, N] field: bit-identical to the whole-field call, other cells untouched."""
    import torch
    w = synth.cfg5(J=6)
    u0 = np.ascontiguousarray(w.u.reshape(20, -1))
    M = P.Model(dict(w.model, m=20))
    full = torch.tensor(u0, device="cuda")
    P.rd_reaction_radau5(full, M, 0.5 * w.dt)
    full = full.cpu().numpy()
    a, b = 301, 3001
    u = torch.tensor(u0, device="cuda")
    P.rd_reaction_radau5_cells(u[:, a:b], M, 0.5 * w.dt)
    got = u.cpu().numpy()
    assert np.array_equal(got[:, a:b], full[:, a:b])
    assert np.array_equal(got[:, :a], u0[:, :a]) and np.array_equal(got[:, b:], u0[:, b:])
    sel = np.random.default_rng(9).choice(u0.shape[1], 500, replace=False).astype(np.int32)
    u = torch.tensor(u0, device="cuda")
    P.rd_reaction_radau5_cells(u, M, 0.5 * w.dt, order=torch.tensor(sel, device="cuda"))
    got = u.cpu().numpy()
    mask = np.zeros(u0.shape[1], dtype=bool)
    mask[sel] = True
    assert np.array_equal(got[:, mask], full[:, mask]) and np.array_equal(got[:, ~mask], u0[:, ~mask])


def test_reaction_cost_keys(P, orc):
    """Keys are the proxy of include/rdmr.h: 64 (log2 sum_i |f_i| / (atol + rtol |y_i|) + 256), clamped
    (FP32 log2 on the device: within one key of a float64 evaluation)."""
    import torch
    u0 = _bz_field(3000, 72)
    spec = dict(kind="oregonator", **synth.OREGONATOR)
    key = P.rd_reaction_cost(torch.tensor(u0, device="cuda"), P.Model(spec)).cpu().numpy()
    Mo = orc.Model(spec)
    s = np.array([np.sum(np.abs(Mo.f(u0[:, c])) / (1e-8 + 1e-8 * np.abs(u0[:, c]))) for c in range(u0.shape[1])])
    ref = np.clip(np.floor((np.log2(s) + 256.0) * 64.0), 0, 65535)
    assert np.abs(key - ref).max() <= 1


def test_species_split_of_diffusion(P):
    """D on species {0, 2} then on {1} equals D on all species, bit for bit (species are independent)."""
    import torch
    w = synth.cfg3(J=8, K=3)
    g1 = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
    g2 = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
    e = list(w.eps_diff)
    g1.diffusion_rock4(e, w.dt)
    g2.diffusion_rock4([e[0], 0.0, e[2]], w.dt)
    g2.diffusion_rock4([0.0, e[1], 0.0], w.dt)
    assert np.array_equal(gpu_leaves(g1)[1], gpu_leaves(g2)[1])


@pytest.mark.parametrize("scheme", [0, 1])
def test_sharded_strang_one_rank_equals_library_step(P, scheme):
    """ShardedStrang on one rank (R through rd_reaction_radau5_cells, D through rd_diffusion_rock4) vs
    rd_strang_step: identical leaves after a step and an adaptation."""
    from paper_1506_04651_b200.shard import GridBackend, ShardedStrang
    w = synth.cfg3(J=8, K=3)
    spec = dict(w.model, m=w.m)
    g1 = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
    g2 = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
    S = ShardedStrang(GridBackend(g2, P.Model(spec)), w.eps_diff)
    for _ in range(2):
        g1.strang_step(P.Model(spec), w.eps_diff, w.dt, scheme)
        S.step(w.dt, scheme)
        k1, u1 = gpu_leaves(g1)
        k2, u2 = gpu_leaves(g2)
        assert np.array_equal(k1, k2) and np.array_equal(u1, u2)
        g1.adapt()
        S.adapt()


def test_emulated_two_rank_reaction(P):
    """The two intervals of a 2-way cost-balanced split, integrated one after the other on one GPU (no
    collectives), reproduce the whole-field reaction bit for bit."""
    import torch
    w = synth.cfg3(J=8, K=3)
    spec = dict(w.model, m=w.m)
    M = P.Model(spec)
    g1 = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
    _, u0 = g1.leaf_tensors()
    ref = u0.clone()
    P.rd_reaction_radau5(ref, M, 0.5 * w.dt)
    u = u0.clone()
    b = P.rd_shard_bounds(u.shape[1], P.rd_reaction_cost(u, M), 2)
    assert 0 < b[1] < u.shape[1]
    for r in range(2):
        P.rd_reaction_radau5_cells(u[:, b[r]:b[r + 1]], M, 0.5 * w.dt)
    assert torch.equal(u, ref)


def _two_rank_worker(rank, world, port, out):
    """One rank of a 2-process ShardedStrang run on the single GPU (gloo collectives, CUDA tensors staged
    through the host): each process owns a replica of the grid, integrates its interval in R and its
    species in D, and exchanges them through torch.distributed."""
    import os
    import torch
    import torch.distributed as dist
    import paper_1506_04651_b200 as P
    from paper_1506_04651_b200.shard import GridBackend, ShardedStrang
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.cfg3(J=8, K=3)
        g = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
        S = ShardedStrang(GridBackend(g, P.Model(dict(w.model, m=w.m))), w.eps_diff)
        res = []
        for scheme in (0, 1):
            S.step(w.dt, scheme)
            k, u = gpu_leaves(g)
            res.append((k.copy(), u.copy(), list(S.last_bounds)))
            S.adapt()
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_sharded_strang_two_ranks_vs_oracle(P, orc):
    """N2 collective path on the GPU: 2 ranks (processes) step one cfg-3-type problem (J = 8) with the
    interval split of R and the species split of D, all-gather / broadcast through torch.distributed.
    Both replicas must be identical bit for bit, and equal to the oracle's Strang step (identical leaf
    set, states within 1e-6 normwise) for RDR then DRD, with an adaptation in between."""
    import torch.multiprocessing as mp
    from tests.test_shard import _free_port
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_two_rank_worker, args=(world, port, out), nprocs=world, join=True)
    w = synth.cfg3(J=8, K=3)
    o = orc.Grid.build(2, w.level_min, w.level_max, w.eps_mr, w.u.reshape(w.m, -1))
    M = orc.Model(dict(w.model, m=w.m))
    for it, scheme in enumerate((0, 1)):
        k0, u0, b0 = out[0][it]
        k1, u1, b1 = out[1][it]
        assert np.array_equal(k0, k1) and np.array_equal(u0, u1) and b0 == b1
        assert len(b0) == 3 and 0 < b0[1] < len(k0)
        assert o.strang(M, w.eps_diff, w.dt, scheme, nthreads=8) == 0
        ok, ou = o.leaves()
        assert np.array_equal(k0, ok)
        err = np.abs(u0 - ou).max(1) / np.abs(ou).max(1)
        assert (err <= 1e-6).all(), (it, err)
        o.set_values(u0)  # continue from the GPU state, as in _strang_parity
        o.adapt()
