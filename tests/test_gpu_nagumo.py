"""GPU parity for SURVEY §8(f) N1: the NAGUMO model and the explicit RK4 reaction option
(reading R-K4) through the C-ABI, against the oracle: rd_reaction_rk4 cell by cell, Radau5 on
NAGUMO (m = 1 thread kernel), and Strang steps with RK4 reactions on an adapting MR grid."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

TOL = 1e-6  # normwise relative, per species (reading S20)


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def _normwise(g, o):
    return np.abs(g - o).max(axis=1) / np.abs(o).max(axis=1)


@pytest.mark.parametrize("nsteps", [1, 3])
def test_rk4_nagumo_cells(P, orc, nsteps):
    import torch
    u0 = synth.random_positive_cells(3001, 1, 61, lo=0.0, hi=1.0)
    spec = dict(kind="nagumo", k=10.0)
    u = torch.tensor(u0, device="cuda")
    P.rd_reaction_rk4(u, P.Model(spec), 5e-3, nsteps)
    o = orc.rk4(u0, orc.Model(spec), 5e-3, nsteps)
    assert np.max(np.abs(u.cpu().numpy() - o)) <= 1e-15  # same arithmetic up to FMA contraction


def test_rk4_bz_cells_short_interval(P, orc):
    """RK4 for the m = 3 model over an interval inside its stability region (h |lambda| < 2.78)."""
    import torch
    u0 = synth.random_bz_cells(500, 62)
    spec = dict(kind="oregonator", **synth.OREGONATOR)
    u = torch.tensor(u0, device="cuda")
    T = 1e-7
    P.rd_reaction_rk4(u, P.Model(spec), T, 2)
    o = orc.rk4(u0, orc.Model(spec), T, 2)
    assert (_normwise(u.cpu().numpy(), o) <= 1e-13).all()


def test_radau5_nagumo_cells(P, orc):
    import torch
    u0 = synth.random_positive_cells(2000, 1, 63, lo=0.0, hi=1.0)
    spec = dict(kind="nagumo", k=10.0)
    u = torch.tensor(u0, device="cuda")
    st = P.rd_stats()
    P.rd_reaction_radau5(u, P.Model(spec), 5e-3, stats=st)
    o, _, ost = orc.radau5(u0, orc.Model(spec), 5e-3, nthreads=8)
    assert (ost == 0).all() and st.n_failed == 0
    assert (_normwise(u.cpu().numpy(), o) <= TOL).all()


def test_rk4_errors(P):
    import torch
    u = torch.zeros((20, 4), dtype=torch.float64, device="cuda")
    spec = dict(kind="mass_action", m=20, reactants=np.array([[0, -1]]), products=np.array([[1, -1]]),
                rate=np.array([1.0]))
    with pytest.raises(P.RdError):
        P.rd_reaction_rk4(u, P.Model(spec), 1e-3)  # m > 4: not supported by the thread form
    with pytest.raises(P.RdError):
        P.rd_reaction_rk4(torch.zeros((1, 4), dtype=torch.float64, device="cuda"), P.Model(dict(kind="nagumo")), 0.0)


@pytest.mark.parametrize("scheme", [0, 1])
def test_strang_nagumo_rk4_mr(P, orc, scheme):
    """Two Strang steps (RDR / DRD) with RK4 reactions on the NAGUMO workload at J = 8, re-adapting after
    each step: identical leaf sets, states within 1e-6 normwise."""
    import torch
    w = synth.cfg6(J=8)
    um = P.mr_rowmajor_to_morton(2, w.level_max, torch.tensor(w.u.reshape(1, -1), device="cuda"))
    g = P.Grid.build(2, w.level_min, w.level_max, w.eps_mr, um)
    o = orc.Grid.build(2, w.level_min, w.level_max, w.eps_mr, w.u.reshape(1, -1))
    gm, om = P.Model(w.model), orc.Model(w.model)
    for it in range(2):
        g.strang_step(gm, w.eps_diff, w.dt, scheme | P.RD_STRANG_RK4)
        assert o.strang(om, w.eps_diff, w.dt, scheme | orc.STRANG_RK4, nthreads=16) == 0
        gk, gu = g.leaf_tensors()
        gk, gu = gk.cpu().numpy().view(np.uint64), gu.cpu().numpy()
        ok, ou = o.leaves()
        assert np.array_equal(gk, ok)
        assert (_normwise(gu, ou) <= TOL).all(), (it, _normwise(gu, ou))
        o.set_values(gu)
        g.set_values(torch.tensor(gu, device="cuda"))
        o.adapt()
        g.adapt()
        gk2, _ = g.leaf_tensors()
        assert np.array_equal(gk2.cpu().numpy().view(np.uint64), o.leaves()[0])
