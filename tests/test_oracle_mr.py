"""Oracle multiresolution (O.6) against brute force, closed forms and invariants."""
import numpy as np
import pytest

import synth
from tests.grids import front_field, leaf_geometry
from tests.mr_ref import DenseTree, tree_from_leaves


def test_threshold_examples():
    """P:589 eps_j = 2^{(d/2)(j-J)} eps; SPEC S:240-242 worked values."""
    eps_j = lambda d, J, eps, j: 2.0 ** ((d / 2) * (j - J)) * eps
    assert eps_j(2, 10, 0.01, 8) == 0.0025
    assert eps_j(3, 9, 1.0, 7) == 0.125
    # the squared form used on both sides: ldexp(eps^2, d (j - J)) == eps_j^2 exactly here
    assert np.ldexp(0.01 * 0.01, 2 * (8 - 10)) == pytest.approx(0.0025 ** 2, rel=1e-15)


def test_prediction_1d_example_via_quadratic_exactness(orc):
    """Eq. inter_1d: (0,1,2) -> (0.75, 1.25) in 1-D; the tensor-product
    prediction is exact for cell averages of quadratics, so a
    quadratic field has zero details and coarsens to L_min everywhere except near
    the mirrored boundary."""
    u = np.array([0.0, 1.0, 2.0])
    pred = (u[1] + (u[0] - u[2]) / 8, u[1] + (u[2] - u[0]) / 8)
    assert pred == (0.75, 1.25)
    J, lmin = 6, 2
    n = 1 << J
    x = (np.arange(n) + 0.5) / n
    yy, xx = np.meshgrid(x, x, indexing="ij")
    h = 1.0 / n
    q = 3 * (xx - 0.5) ** 2 + (yy - 0.5) ** 2 + (4 * h * h / 12)  # cell averages of a quadratic
    g = orc.Grid.build(2, lmin, J, 1e-6, q[None])
    keys, _ = g.leaves()
    lv, cen, _ = leaf_geometry(2, keys)
    inner = np.all((cen > 0.3) & (cen < 0.7), axis=1)
    assert lv[inner].max() <= lmin + 1  # (the boundary band + radius-2 grading keeps level lmin+1)


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
