"""Oracle two-point-flux operator (the App. A setting where every coefficient follows
from the link type and the level; reading R-T), pinned to what the definition
fixes: the uniform-grid reduction, constants in the kernel, conservation and volume-weighted symmetry
(a two-point flux is one number per face), negative semi-definiteness, the Gershgorin bound, and the
coefficient values across a level jump (face area over centre distance 1.5 h_fine)."""
import numpy as np
import pytest

from tests.grids import front_field, leaf_geometry


def _grid(orc, dim, lmin, J, eps, mode):
    u = front_field(dim, J, 1)
    g = orc.Grid.build(dim, lmin, J, eps, u.reshape(1, -1))
    g.set_operator(mode)
    return g


def _dense(g):
    n = g.n_leaves
    return np.stack([g.apply(np.eye(n)[k]) for k in range(n)], axis=1)  # column k = A e_k


@pytest.mark.parametrize("dim,J", [(2, 5), (3, 3)])
def test_uniform_grid_reduction(orc, dim, J):
    a, b = _grid(orc, dim, J, J, 0.0, 0), _grid(orc, dim, J, J, 0.0, 1)
    x = np.random.default_rng(1).standard_normal(a.n_leaves)
    assert np.array_equal(a.apply(x), b.apply(x))
    assert a.rho1 == b.rho1 == 4 * dim * 4.0 ** J


@pytest.mark.parametrize("dim,lmin,J,eps", [(2, 2, 6, 1e-2), (3, 1, 4, 1e-2)])
def test_conservation_symmetry_definiteness(orc, dim, lmin, J, eps):
    g = _grid(orc, dim, lmin, J, eps, 1)
    keys, _ = g.leaves()
    levels = np.array([int(k) >> 58 for k in keys])
    assert levels.min() < levels.max()  # the case has level jumps
    vol = 2.0 ** (-dim * levels)
    rng = np.random.default_rng(2)
    x, z = rng.standard_normal(g.n_leaves), rng.standard_normal(g.n_leaves)
    ax, az = g.apply(x), g.apply(z)
    assert np.abs(g.apply(np.ones(g.n_leaves))).max() <= 1e-9 * g.rho1
    assert abs((vol * ax).sum()) <= 1e-12 * (vol * np.abs(ax)).sum()
    assert abs((vol * z * ax).sum() - (vol * x * az).sum()) <= 1e-12 * (vol * np.abs(z * ax)).sum()
    assert (vol * x * ax).sum() < 0.0


def test_gershgorin_and_spectrum(orc):
    g = _grid(orc, 2, 2, 5, 1e-2, 1)
    A = _dense(g)
    assert np.abs(np.diag(A) * 2).max() == pytest.approx(g.rho1, rel=1e-15)  # row sum = 2 |diag|
    assert np.abs(np.linalg.eigvals(A)).max() <= g.rho1 * (1 + 1e-12)
    assert (np.linalg.eigvals(A).real <= 1e-9 * g.rho1).all()


def test_level_jump_coefficients(orc):
    """Across a face between a level-j leaf F and a level-(j-1) leaf L: A[F, L] = 4^j / 1.5 and
    A[L, F] = 4^j / (1.5 2^d) (flux |face| (u_L - u_F) / (1.5 h_j), divided by the cell volume)."""
    dim = 2
    g = _grid(orc, dim, 2, 6, 1e-2, 1)
    keys, _ = g.leaves()
    lv, cen, vol = leaf_geometry(dim, keys)
    A = _dense(g)
    found = 0
    for f in range(len(keys)):
        for l in np.nonzero(A[f])[0]:
            if lv[l] != lv[f] - 1:
                continue
            j = lv[f]
            assert A[f, l] == 4.0 ** j / 1.5
            assert A[l, f] == 4.0 ** j / (1.5 * 2 ** dim)
            d = np.abs(cen[l] - cen[f])
            assert sorted(d)[-1] == pytest.approx(1.5 * 2.0 ** -j)  # centre distance along the normal
            found += 1
    assert found > 0
