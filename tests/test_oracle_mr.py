"""Oracle multiresolution (O.6) against brute force, closed forms and invariants."""
import numpy as np
import pytest

import synth
from tests.grids import front_field, leaf_geometry
from tests.mr_ref import DenseTree, tree_from_leaves


def test_threshold_examples(orc):
    """P:589 eps_j = 2^{(d/2)(j-J)} eps, through the oracle's own E_j = eps_j^2; SPEC S:240-242 worked
    values (eps_8 = 0.0025 at d = 2, J = 10, eps = 0.01; eps_7 = 0.125 at d = 3, J = 9, eps = 1)."""
    assert orc.threshold_sq(2, 10, 0.01, 8) == pytest.approx(0.0025 ** 2, rel=1e-15)
    assert orc.threshold_sq(3, 9, 1.0, 7) == 0.125 ** 2
    assert orc.threshold_sq(2, 10, 0.01, 10) == 0.01 * 0.01  # the finest level carries eps itself
    # one level coarser divides eps_j by 2^{d/2}: E_j by 2^d, exactly
    for d in (2, 3):
        for j in range(1, 10):
            assert orc.threshold_sq(d, 10, 0.3, j - 1) * 2 ** d == orc.threshold_sq(d, 10, 0.3, j)


def test_prediction_1d_example(orc):
    """Eq. inter_1d through the oracle's tensor-product prediction: values constant along y
    (and z) reduce it to the 1-D rule, (0, 1, 2) -> (0.75, 1.25) for the two children."""
    u = np.array([0.0, 1.0, 2.0])
    v2 = np.tile(u, 3)  # index oy*3 + ox
    assert orc.predict_vals(2, v2, (0, 0)) == 0.75 and orc.predict_vals(2, v2, (1, 1)) == 1.25
    v3 = np.tile(u, 9)
    assert orc.predict_vals(3, v3, (0, 1, 0)) == 0.75 and orc.predict_vals(3, v3, (1, 0, 1)) == 1.25
    # along y: the same example, child bit of y decides
    vy = np.repeat(u, 3)
    assert orc.predict_vals(2, vy, (1, 0)) == 0.75 and orc.predict_vals(2, vy, (0, 1)) == 1.25


def _avg_pow(p, a, b):
    """Average of x^p over [a, b] (exact for the dyadic inputs used here)."""
    return (b ** (p + 1) - a ** (p + 1)) / ((p + 1) * (b - a))


@pytest.mark.parametrize("px,py", [(0, 0), (1, 0), (0, 1), (2, 0), (0, 2), (1, 1), (2, 2)])
def test_prediction_exact_on_tensor_quadratics(orc, px, py):
    """the 3rd-order centred prediction reproduces cell averages of polynomials of degree
    <= 2 per direction (tensor product).  Parent cells [-1.5,-0.5], [-0.5,0.5], [0.5,1.5];
    children of the centre cell [-0.5,0], [0,0.5]."""
    par = [(-1.5, -0.5), (-0.5, 0.5), (0.5, 1.5)]
    ch = [(-0.5, 0.0), (0.0, 0.5)]
    v = np.array([[_avg_pow(px, *par[ox]) * _avg_pow(py, *par[oy]) for ox in range(3)] for oy in range(3)])
    for bx in (0, 1):
        for by in (0, 1):
            want = _avg_pow(px, *ch[bx]) * _avg_pow(py, *ch[by])
            assert orc.predict_vals(2, v, (bx, by)) == pytest.approx(want, abs=1e-15)
    # a cubic is NOT reproduced (the rule is 3rd order, not 4th): guards against a wrong stencil weight
    v3 = np.array([[_avg_pow(3, *par[ox]) for ox in range(3)] for oy in range(3)])
    assert abs(orc.predict_vals(2, v3, (0, 0)) - _avg_pow(3, *ch[0])) > 1e-3


def _tie_field(J, amp, lvl):
    """Constant 0.5 at level J except one level-`lvl` parent (the cell at (2, 2) of level lvl - 1) whose
    4 children at level lvl carry 0.5 + amp * (+1, -1, -1, +1): parent averages stay 0.5, every
    prediction is exactly 0.5, and those 4 children have detail +-amp, i.e. Q = amp^2 (s_i = 1)."""
    n = 1 << J
    u = np.full((1, n, n), 0.5)
    c = 1 << (J - lvl)  # level-J cells per level-lvl cell
    sgn = {(0, 0): 1.0, (1, 0): -1.0, (0, 1): -1.0, (1, 1): 1.0}
    for (bx, by), s in sgn.items():
        x0, y0 = (4 + bx) * c, (4 + by) * c
        u[0, y0:y0 + c, x0:x0 + c] = 0.5 + s * amp
    return u


@pytest.mark.parametrize("strict", [True, False])
def test_coarsen_threshold_tie(orc, strict):
    """P:590-596 / reading S12: a node is coarsened when its children's details are SMALLER than the
    threshold.  Q = E_J exactly (eps = 2^-4, amp = 2^-4, Q = 2^-8 = E_J) must keep the finest cells;
    an amplitude one part in 2^20 smaller coarsens them."""
    J, eps = 5, 2.0 ** -4
    amp = 2.0 ** -4 if strict else 2.0 ** -4 * (1 - 2.0 ** -20)
    assert amp * amp <= orc.threshold_sq(2, J, eps, J)
    g = orc.Grid.build(2, 1, J, eps, _tie_field(J, amp, J))
    keys, _ = g.leaves()
    lv = keys >> np.uint64(58)
    assert (lv == J).any() == strict


@pytest.mark.parametrize("tie", [True, False])
def test_refine_threshold_tie(orc, tie):
    """P:590-596 / reading S12: a leaf is refined when its detail EXCEEDS the threshold.  Leaves at level
    J-1 = L_min with Q = E_{J-1} exactly (amp = 2^-5, eps = 2^-4: Q = 2^-10 = E_{J-1}) stay; one part
    in 2^20 more refines them."""
    J, eps = 5, 2.0 ** -4
    amp = 2.0 ** -5 if tie else 2.0 ** -5 * (1 + 2.0 ** -20)
    g = orc.Grid.build(2, J - 1, J, eps, _tie_field(J, amp, J - 1))
    keys, _ = g.leaves()
    assert ((keys >> np.uint64(58)) == J - 1).all()  # the build sits on the L_min floor
    g.adapt()
    keys, _ = g.leaves()
    assert ((keys >> np.uint64(58)) == J).any() == (not tie)


def test_eps_zero_is_uniform_finest(orc):
    J = 5
    u = front_field(2, J, m=2)
    g = orc.Grid.build(2, 2, J, 0.0, u)
    keys, vals = g.leaves()
    assert len(keys) == 4 ** J and all((int(k) >> 58) == J for k in keys)
    # values are the input re-ordered in Morton order (bit-for-bit)
    for r, key in enumerate(keys[:200]):
        lev, k = orc.key_decode(2, int(key))
        assert vals[0, r] == u[0, k[1], k[0]] and vals[1, r] == u[1, k[1], k[0]]


@pytest.mark.parametrize("dim,J,lmin,eps", [(2, 5, 2, 1e-2), (2, 6, 2, 3e-3), (3, 4, 1, 1e-2), (3, 4, 2, 3e-3)])
def test_build_matches_brute_force(orc, dim, J, lmin, eps):
    u = front_field(dim, J, m=3)
    g = orc.Grid.build(dim, lmin, J, eps, u)
    ko, uo = g.leaves()
    b = DenseTree.build(dim, lmin, J, eps, u, seed=5)  # random sequential collapse order
    kb, ub = b.leaves()
    assert np.array_equal(ko, kb)
    assert np.array_equal(uo, ub)
    assert g.check() == 0


@pytest.mark.parametrize("dim,J,lmin,eps", [(2, 5, 2, 1e-2), (2, 6, 3, 3e-3), (3, 4, 1, 1e-2)])
def test_adapt_matches_brute_force_and_conserves(orc, dim, J, lmin, eps):
    g = orc.Grid.build(dim, lmin, J, eps, front_field(dim, J, m=3))
    ko, uo = g.leaves()
    for it in range(2):
        u2 = uo.copy()
        u2[0] = uo[0] + 0.3 * np.sin(0.37 * np.arange(len(ko)) + it)  # rough perturbation -> refinement
        g.set_values(u2)
        b = tree_from_leaves(dim, lmin, J, eps, ko, u2)
        g.adapt()
        ka, ua = g.leaves()
        b.adapt(seed=11 + it)
        kb, ub = b.leaves()
        assert np.array_equal(ka, kb) and np.array_equal(ua, ub)
        assert g.check() == 0
        _, _, v0 = leaf_geometry(dim, ko)
        _, _, v1 = leaf_geometry(dim, ka)
        for i in range(3):
            assert abs((v0 * u2[i]).sum() - (v1 * ua[i]).sum()) <= 1e-14 * np.abs(v0 * u2[i]).sum()
        ko, uo = ka, ua


def test_adapt_of_unchanged_field_is_stable(orc):
    """Re-adapting values that the tree already resolves neither refines (details
    below eps) nor loses accuracy: leaf values of unchanged leaves are untouched."""
    g = orc.Grid.build(2, 2, 6, 1e-2, front_field(2, 6, m=1))
    k0, u0 = g.leaves()
    g.adapt()
    k1, u1 = g.leaves()
    common = np.intersect1d(k0, k1)
    i0 = np.searchsorted(k0, common)
    i1 = np.searchsorted(k1, common)
    assert np.array_equal(u0[:, i0], u1[:, i1])


def test_cfg3_leaf_count_in_configured_range(orc):
    """BJ configs[2]: 'roughly 10^5 to 2x10^5 leaves'."""
    w = synth.cfg3()
    g = orc.Grid.build(2, w.level_min, w.level_max, w.eps_mr, w.u)
    n = g.n_leaves
    assert 1e5 <= n <= 2.5e5, n
    assert g.check() == 0
