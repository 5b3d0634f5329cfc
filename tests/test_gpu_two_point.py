"""GPU parity for SURVEY §8(f) N4: the two-point-flux leaf operator (App. A; DESIGN.md
reading R-T) in its explicit-weight form (RD_OP_TWO_POINT) and App. A's compact storage
(RD_OP_TWO_POINT_COMPACT: column + link type, coefficient rebuilt from the level), against the oracle's
set_operator(1): y = A x, the Gershgorin bound rho1, controlled Rock4, and Strang steps with
re-adaptation (the operator choice persists through mr_adapt)."""
import numpy as np
import pytest

import synth
from tests.grids import front_field
from tests.test_gpu_mr_rock4 import assert_same_grid, gpu_build, gpu_leaves

pytestmark = pytest.mark.gpu

MODES = [1, 2]  # RD_OP_TWO_POINT, RD_OP_TWO_POINT_COMPACT
CASES = [(2, 2, 6, 1e-2, 1), (2, 3, 7, 3e-3, 3), (2, 0, 5, 5e-2, 2), (3, 1, 4, 1e-2, 1), (3, 2, 5, 2e-2, 2)]


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def _pair(P, orc, dim, lmin, J, eps, m, mode):
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    g.set_operator(mode)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    o.set_operator(1)
    return g, o


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dim,lmin,J,eps,m", CASES)
def test_two_point_apply(P, orc, dim, lmin, J, eps, m, mode):
    import torch
    g, o = _pair(P, orc, dim, lmin, J, eps, m, mode)
    assert g.info()["rho1"] == o.rho1
    x = np.random.default_rng(11).standard_normal(g.n_leaves)
    y = g.fv_apply(torch.tensor(x, device="cuda")).cpu().numpy()
    yo = o.apply(x)
    assert np.max(np.abs(y - yo)) <= 1e-12 * np.abs(yo).max()
    # a two-point operator annihilates constants exactly up to rounding of the row (explicit diagonal
    # = -sum of the row, or the compact form's differences x_c - x_r = 0)
    one = g.fv_apply(torch.ones(g.n_leaves, dtype=torch.float64, device="cuda")).cpu().numpy()
    if mode == 2:
        assert not one.any()
    else:
        assert np.abs(one).max() <= 1e-13 * o.rho1


def test_compact_equals_explicit(P, orc):
    """The compact form rebuilds every coefficient from (type, level): same operator as the explicit
    weights to rounding (the diagonal is folded into differences instead of a stored weight)."""
    import torch
    u = front_field(2, 8, 1)
    g = gpu_build(P, 2, 2, 8, 5e-3, u)
    x = torch.tensor(np.random.default_rng(12).standard_normal(g.n_leaves), device="cuda")
    g.set_operator(1)
    a = g.fv_apply(x).cpu().numpy()
    g.set_operator(2)
    b = g.fv_apply(x).cpu().numpy()
    assert np.max(np.abs(a - b)) <= 1e-13 * np.abs(a).max()


def test_mode_switch_back_to_prediction(P, orc):
    """mr_set_operator(0) restores the prediction operator (identical to a grid that never switched)."""
    import torch
    dim, lmin, J, eps = 2, 2, 6, 1e-2
    u = front_field(dim, J, 1)
    g, h = gpu_build(P, dim, lmin, J, eps, u), gpu_build(P, dim, lmin, J, eps, u)
    x = torch.tensor(np.random.default_rng(13).standard_normal(g.n_leaves), device="cuda")
    ref = h.fv_apply(x).cpu().numpy()
    g.set_operator(2)
    assert not np.array_equal(g.fv_apply(x).cpu().numpy(), ref)
    g.set_operator(0)
    assert np.array_equal(g.fv_apply(x).cpu().numpy(), ref)
    assert g.info()["rho1"] == h.info()["rho1"]


def test_set_operator_errors(P):
    import torch
    L = P.lib()
    u = torch.zeros((1, 4 ** 5), dtype=torch.float64, device="cuda")
    g = P.Grid.build(2, 1, 5, 0.0, u)
    assert L.mr_set_operator(g.h, 3, None) == P.RD_EINVAL
    assert L.mr_set_operator(g.h, -1, None) == P.RD_EINVAL
    assert L.mr_set_operator(None, 1, None) == P.RD_EINVAL


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dim,lmin,J,eps,T", [(2, 3, 7, 3e-3, 1e-3), (2, 2, 6, 1e-2, 1e-2), (3, 2, 5, 2e-2, 1e-3)])
def test_two_point_rock4(P, orc, dim, lmin, J, eps, T, mode, monkeypatch):
    """Controlled Rock4 with the two-point operator (always the assembled kernel, also in 3-D and when
    the matrix-free form is requested): normwise relative error <= 1e-6, mass conserved."""
    monkeypatch.setenv("RDMR_R4_MODE", "free")  # ignored for two-point operators
    m = 3
    g, o = _pair(P, orc, dim, lmin, J, eps, m, mode)
    epsd = [2.5e-3, 2.5e-3, 1.5e-3]
    st = P.rd_stats()
    g.diffusion_rock4(epsd, T, stats=st)
    o.diffuse(epsd, T)
    gk, gu = gpu_leaves(g)
    _, ou = o.leaves()
    err = np.abs(gu - ou).max(1) / np.abs(ou).max(1)
    assert (err <= 1e-6).all(), err
    assert st.rock4_mat_slots >= len(gk)
    vol = np.array([2.0 ** (-dim * (int(k) >> 58)) for k in gk])
    _, u0 = o.leaves()
    assert np.allclose((gu * vol).sum(1), (ou * vol).sum(1), rtol=1e-12)


@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("which", ["2d", "3d"])
def test_two_point_strang_adapt(P, orc, mode, which, scheme):
    """Two Strang steps (BZ, Radau5 + Rock4) with re-adaptation after each: identical leaf sets,
    states within 1e-6 normwise; the operator mode survives mr_adapt on both sides."""
    import torch
    w = synth.cfg3(J=8, K=3) if which == "2d" else synth.cfg4(J=5, K=3)
    g = gpu_build(P, w.dim, w.level_min, w.level_max, w.eps_mr, w.u)
    o = orc.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, w.u.reshape(w.m, -1))
    g.set_operator(mode)
    o.set_operator(1)
    spec = dict(w.model, m=w.m)
    gm, om = P.Model(spec), orc.Model(spec)
    for it in range(2):
        g.strang_step(gm, w.eps_diff, w.dt, scheme)
        assert o.strang(om, w.eps_diff, w.dt, scheme, nthreads=16) == 0
        gk, gu = gpu_leaves(g)
        ok, ou = o.leaves()
        assert np.array_equal(gk, ok)
        err = np.abs(gu - ou).max(1) / np.abs(ou).max(1)
        assert (err <= 1e-6).all(), (it, err)
        o.set_values(gu)
        g.set_values(torch.tensor(gu, device="cuda"))
        o.adapt()
        g.adapt()
        assert_same_grid(g, o)
        assert g.info()["rho1"] == o.rho1
