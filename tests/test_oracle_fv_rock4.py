"""Oracle FV operator (O.5) and Rock4 (O.4) against closed forms and library routines."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.linalg import expm_multiply
from scipy.special import roots_chebyt

from oracle import rock4_family
from tests.grids import front_field, leaf_geometry


def _uniform(orc, dim, J, m=1):
    n = 1 << J
    return orc.Grid.build(dim, J, J, 0.0, np.zeros((m,) + (n,) * dim))


def _neumann_laplacian_morton(dim, J, keys):
    """Textbook 5/7-point cell-centred Neumann Laplacian, assembled by brute force."""
    from tests.mr_ref import morton_decode
    n = 1 << J
    idx = {morton_decode(dim, int(k))[1]: r for r, k in enumerate(keys)}
    rows, cols, vals = [], [], []
    for k, r in idx.items():
        for a in range(dim):
            for s in (-1, 1):
                q = list(k)
                q[a] += s
                if 0 <= q[a] < n:
                    rows += [r, r]
                    cols += [idx[tuple(q)], r]
                    vals += [n * n, -n * n]
    return sp.csr_matrix((vals, (rows, cols)), shape=(len(keys),) * 2)


@pytest.mark.parametrize("dim,J", [(2, 5), (3, 3)])
def test_uniform_operator_is_textbook_stencil(orc, dim, J):
    g = _uniform(orc, dim, J)
    keys, _ = g.leaves()
    A = _neumann_laplacian_morton(dim, J, keys)
    x = np.random.default_rng(0).normal(size=len(keys))
    assert np.allclose(g.apply(x), A @ x, rtol=1e-14, atol=1e-10)
    assert g.rho1 == 4 * dim * 4.0 ** J  # Gershgorin 4d/h^2


def test_gershgorin_paper_magnitude(orc):
    """h = 1/1024 in 2-D, eps = 2.5e-3 -> largest eigenvalues about -2e4."""
    rho = 4 * 2 * 1024.0 ** 2 * 2.5e-3
    assert rho == 20971.52
    assert 1.5e4 < rho < 2.5e4
    assert _uniform(orc, 2, 7).rho1 * 2.5e-3 == 327.68  # cfg 1


@pytest.mark.parametrize("dim,J,lmin", [(2, 7, 3), (3, 5, 2)])
def test_adaptive_operator_properties(orc, dim, J, lmin):
    g = orc.Grid.build(dim, lmin, J, 1e-2, front_field(dim, J))
    keys, _ = g.leaves()
    lv, cen, vol = leaf_geometry(dim, keys)
    assert len(set(lv)) >= 3  # genuinely adaptive
    assert np.abs(g.apply(np.ones(len(keys)))).max() == 0.0
    x = np.sin(7 * cen[:, 0]) + cen[:, 1] ** 3
    assert abs((vol * g.apply(x)).sum()) <= 1e-13 * np.abs(vol * g.apply(x)).sum()  # conservation
    # exact for cell averages of quadratics away from the boundary (ghost prediction exact for degree 2)
    h = 2.0 ** -lv
    q = (cen ** 2).sum(1) + dim * h ** 2 / 12
    inner = np.all((cen > 0.2) & (cen < 0.8), axis=1)
    assert np.abs(g.apply(q)[inner] - 2 * dim).max() < 1e-9


def test_rock4_table_structure(orc):
    for s in (5, 6, 7, 8, 12, 30, 80, 150):
        c = orc.rock4_coeffs(s)
        assert np.allclose(c["nu"] + c["kappa"], 1.0, atol=1e-12)
        z = np.array([-0.1, -0.05, -0.025])
        R = rock4_family.eval_w(c["sigma"], z) * rock4_family.eval_P(c["mu"], c["nu"], c["kappa"], z)
        err = np.abs(R - np.exp(z))
        assert err[0] / err[1] > 25 and err[1] / err[2] > 25  # R - e^z = O(z^5): order 4
        zz = -c["ell"] * np.random.default_rng(s).uniform(0, 1, 200000)
        Rz = rock4_family.eval_w(c["sigma"], zz) * rock4_family.eval_P(c["mu"], c["nu"], c["kappa"], zz)
        assert np.abs(Rz).max() <= 1.0 + 1e-6  # stable on [-ell_s, 0] (sampled criterion, O.4 K1)


def test_rock4_orthogonality_independent_quadrature(orc):
    """P_n is orthogonal for w(z)^2 / sqrt(1 - x^2) on [-1, 1] (checked with scipy's
    Gauss-Chebyshev rule, not the generator's)."""
    for s in (7, 20, 60):
        c = orc.rock4_coeffs(s)
        x, wq = roots_chebyt(3 * s + 10)
        z = (x - 1.0) * c["ell"] / 2.0
        Pn = rock4_family.eval_P(c["mu"], c["nu"], c["kappa"], z)
        w2 = rock4_family.eval_w(c["sigma"], z) ** 2
        for k in range(s - 4):
            Tk = np.cos(k * np.arccos(x))
            terms = wq * w2 * Pn * Tk
            assert abs(terms.sum()) <= 1e-11 * np.abs(terms).sum()  # zero up to cancellation


def test_rock4_ell_growth(orc):
    """Stability interval grows like s^2; survey probe values."""
    probe = {5: 6.0535, 6: 9.9421, 7: 14.533, 8: 19.833, 9: 25.843, 10: 32.562, 12: 48.126, 16: 87.753, 32: 359.52}
    for s, ell in probe.items():
        assert abs(orc.rock4_coeffs(s)["ell"] - ell) <= 2e-4 * ell
    r = orc.rock4_coeffs(150)["ell"] / 150 ** 2
    assert 0.34 < r < 0.36


def _eigenmode(dim, J, keys, kvec):
    from tests.mr_ref import morton_decode
    n = 1 << J
    v = np.ones(len(keys))
    for r, key in enumerate(keys):
        k = morton_decode(dim, int(key))[1]
        for a in range(dim):
            v[r] *= np.cos(np.pi * kvec[a] * (k[a] + 0.5) / n)
    lam = -(4.0 * n * n) * sum(np.sin(np.pi * kk / (2 * n)) ** 2 for kk in kvec)
    return v, lam


@pytest.mark.parametrize("s", [5, 9, 20])
def test_rock4_forced_step_on_eigenmode(orc, s):
    """Single step on a Neumann eigenmode: x_{n+1} = R_s(h eps lambda) v (closed form)."""
    J = 6
    g = _uniform(orc, 2, J)
    keys, _ = g.leaves()
    v, lam = _eigenmode(2, J, keys, (3, 5))
    eps = 2.5e-3
    c = orc.rock4_coeffs(s)
    h = 0.7 * c["ell"] / (eps * g.rho1)
    out, e = g.rock4_forced(v, eps, h, s)
    z = h * eps * lam
    Rz = rock4_family.eval_w(c["sigma"], z) * rock4_family.eval_P(c["mu"], c["nu"], c["kappa"], np.array([z]))[0]
    tol = 1e-12 * s * s  # rounding growth through the s-stage recurrence
    assert np.abs(out - Rz * v).max() <= tol
    Pz = rock4_family.eval_P(c["mu"], c["nu"], c["kappa"], np.array([z]))[0]
    assert np.abs(e - c["sigma"][3] * z ** 4 * Pz * v).max() <= tol * (1 + abs(c["sigma"][3] * z ** 4))


def test_rock4_adaptive_vs_exact_decay(orc):
    J = 7
    g = _uniform(orc, 2, J)
    keys, _ = g.leaves()
    v, lam = _eigenmode(2, J, keys, (2, 1))
    for T in (1e-3, 1e-2):
        x, st = g.rock4(v, 2.5e-3, T)
        assert np.abs(x - np.exp(2.5e-3 * lam * T) * v).max() <= 1e-7
        assert st["steps"] >= 1


@pytest.mark.parametrize("dim,J,lmin", [(2, 6, 2), (3, 4, 1)])
def test_rock4_adaptive_grid_vs_expm_multiply(orc, dim, J, lmin):
    g = orc.Grid.build(dim, lmin, J, 1e-2, front_field(dim, J))
    keys, u = g.leaves()
    N = len(keys)
    A = np.column_stack([g.apply(np.eye(N)[:, i]) for i in range(N)])  # assembled by probing
    eps, T = 2.5e-3, 2e-3
    x, st = g.rock4(u[0], eps, T)
    ref = expm_multiply(sp.csr_matrix(eps * T * A), u[0])
    assert np.abs(x - ref).max() <= 1e-6 * np.abs(ref).max()
    _, _, vol = leaf_geometry(dim, keys)
    assert abs((vol * x).sum() - (vol * u[0]).sum()) <= 1e-13 * abs((vol * u[0]).sum())
    # Gershgorin bound really bounds the spectrum
    assert np.abs(np.linalg.eigvals(A)).max() <= g.rho1 * (1 + 1e-12)


@pytest.mark.parametrize("dim,J,lmin", [(2, 6, 2), (3, 4, 1)])
def test_rock4_warm_start_consecutive_substeps_vs_expm_multiply(orc, dim, J, lmin):
    """Reading R-K5b: consecutive D substeps on one grid start each species' controller from the step size
    it proposed when the previous substep ended (h0 = T on a fresh grid).  Three substeps of T must still
    give exp(3 T eps A) u0 (expm_multiply) within the tolerance-derived bound, and the warm-started
    substeps must reject fewer steps than the cold first one."""
    g = orc.Grid.build(dim, lmin, J, 1e-2, front_field(dim, J))
    keys, u = g.leaves()
    N = len(keys)
    A = np.column_stack([g.apply(np.eye(N)[:, i]) for i in range(N)])
    eps, T = 2.5e-3, 3e-2  # long enough that the cold h0 = T is rejected
    rej = []
    for _ in range(3):
        rej.append(g.diffuse([eps], T)["rejects"])
    _, x = g.leaves()
    ref = expm_multiply(sp.csr_matrix(3 * eps * T * A), u[0])
    assert np.abs(x[0] - ref).max() <= 1e-6 * np.abs(ref).max()
    assert rej[0] >= 1 and rej[1] < rej[0] and rej[2] < rej[0], rej
