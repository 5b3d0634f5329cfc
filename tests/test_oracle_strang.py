"""Oracle Strang step (O.7): degenerate cases reduce to the sub-solvers."""
import numpy as np
import pytest

import synth
from tests.grids import front_field


def test_no_reaction_equals_diffusion(orc):
    zero = dict(kind="mass_action", m=3, reactants=np.array([[0, -1]]), products=np.array([[-1, -1]]),
                rate=np.array([0.0]))
    model = orc.Model(zero)
    eps = np.array([2.5e-3, 2.5e-3, 1.5e-3])
    u = front_field(2, 6, m=3)
    g1 = orc.Grid.build(2, 2, 6, 1e-2, u)
    g2 = orc.Grid.build(2, 2, 6, 1e-2, u)
    assert g1.strang(model, eps, 1e-3, scheme=0) == 0
    g2.diffuse(eps, 1e-3)
    assert np.allclose(g1.leaves()[1], g2.leaves()[1], rtol=0, atol=1e-10)


def test_no_diffusion_equals_reaction(orc):
    model = orc.Model(dict(kind="oregonator"))
    w = synth.cfg1(J=5)
    g = orc.Grid.build(2, 5, 5, 0.0, w.u)
    k, u0 = g.leaves()
    for scheme in (0, 1):
        g.set_values(u0)
        assert g.strang(model, np.zeros(3), 1e-3, scheme=scheme) == 0
        ref, _, st = orc.radau5(u0, model, 1e-3)
        got = g.leaves()[1]
        for i in range(3):
            assert np.abs(got[i] - ref[i]).max() <= 1e-6 * np.abs(ref[i]).max()


def test_rdr_and_drd_agree_to_splitting_error(orc):
    model = orc.Model(dict(kind="oregonator"))
    w = synth.cfg1(J=5)
    eps = np.array(w.eps_diff)
    outs = []
    for scheme in (0, 1):
        g = orc.Grid.build(2, 5, 5, 0.0, w.u)
        assert g.strang(model, eps, 1e-4, scheme=scheme) == 0
        outs.append(g.leaves()[1])
    for i in range(3):
        assert np.abs(outs[0][i] - outs[1][i]).max() <= 1e-3 * np.abs(outs[0][i]).max()


def _strang_run(orc, model, w, eps, T, n, scheme, tol, lie=False):
    g = orc.Grid.build(2, 5, 5, 0.0, w.u)
    dt = T / n
    for _ in range(n):
        if lie:  # the first-order Lie split R_dt o D_dt, the negative control of the order test
            g.diffuse(eps, dt, rtol=tol, atol=tol)
            g.react(model, dt, rtol=tol, atol=tol)
        else:
            assert g.strang(model, eps, dt, scheme=scheme, krtol=tol, katol=tol, rtol=tol, atol=tol) == 0
    return g.leaves()[1]


def _order(orc, scheme, lie=False):
    model = orc.Model(dict(kind="oregonator"))
    w = synth.cfg1(J=5)
    eps = np.array(w.eps_diff)
    T, tol, ns = 8e-4, 1e-11, (2, 4, 8, 16)
    ref = _strang_run(orc, model, w, eps, T, 128, scheme, tol, lie)
    errs = []
    for n in ns:
        u = _strang_run(orc, model, w, eps, T, n, scheme, tol, lie)
        errs.append(max(np.abs(u[i] - ref[i]).max() / np.abs(ref[i]).max() for i in range(3)))
    return np.polyfit(np.log(T / np.array(ns)), np.log(errs), 1)[0], errs


@pytest.mark.parametrize("scheme", [0, 1])
def test_strang_order_two(orc, scheme):
    """P:351-363 (§2.1): both Strang compositions (RDR default, DRD) are second order in dt.  cfg 1 at
    J = 5, T = 8e-4 in n = 2, 4, 8, 16 steps against 128 steps, sub-solver tolerances 1e-11 (far below
    the splitting error): the log-log slope is 2 +- 0.3.  A wrong composition (a dropped half step, the
    substeps in Lie order, a full dt reaction on both sides) makes it first order or inconsistent."""
    slope, errs = _order(orc, scheme)
    assert abs(slope - 2.0) <= 0.3, (slope, errs)
    assert errs[-1] < 2e-5


def test_lie_split_is_first_order_control(orc):
    """Negative control for test_strang_order_two: the Lie composition on the same stiff BZ problem
    shows a slope well below 2 (about 1.3 here: first order, with the stiff transient), so the order
    test discriminates a Lie split from a Strang one."""
    slope, errs = _order(orc, 0, lie=True)
    assert slope < 1.6, (slope, errs)
