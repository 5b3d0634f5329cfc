"""Oracle Strang step (O.7): degenerate cases reduce to the sub-solvers."""
import numpy as np

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
