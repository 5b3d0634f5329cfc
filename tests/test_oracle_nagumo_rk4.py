"""Oracle NAGUMO model and RK4 reaction option (DESIGN.md reading
R-K4) pinned to closed forms: the model's values and extrema, RK4's stability polynomial on a linear
ODE, order 4 against the exact implicit solution of u' = k u^2 (1 - u), and the Strang reductions."""
import math

import numpy as np
import pytest

import synth
from tests.grids import front_field

K = 10.0


def _nag(orc, k=K):
    return orc.Model(dict(kind="nagumo", k=k))


def test_nagumo_closed_form(orc):
    """f(u) = k u^2 (1 - u): zeros at 0 and 1, f(1/2) = k/8, maximum 4k/27 at u = 2/3 where
    f' = k (2u - 3u^2) vanishes; |f'| <= 3k on [0, 1]."""
    M = _nag(orc)
    assert M.f([0.0])[0] == 0.0 and M.f([1.0])[0] == 0.0
    assert M.f([0.5])[0] == K / 8
    assert M.f([2.0 / 3.0])[0] == pytest.approx(4 * K / 27, rel=1e-15)
    assert abs(M.jac([2.0 / 3.0])[0, 0]) <= 1e-14
    for u in np.linspace(0.0, 1.0, 101):
        h = 1e-6
        fd = (M.f([u + h])[0] - M.f([u - h])[0]) / (2 * h)
        assert M.jac([u])[0, 0] == pytest.approx(fd, rel=1e-7, abs=1e-7)
        assert abs(M.jac([u])[0, 0]) <= 3 * K


def test_rk4_stability_polynomial(orc):
    """One RK4 step on y' = -lam y gives R(z) = 1 + z + z^2/2 + z^3/6 + z^4/24 exactly, z = -h lam."""
    spec = dict(kind="mass_action", m=1, reactants=np.array([[0, -1]]), products=np.array([[-1, -1]]),
                rate=np.array([1.0]))
    M = orc.Model(spec)
    for z in (-0.1, -0.5, -1.0, -2.5):
        y = orc.rk4(np.ones((1, 1)), M, -z, 1)[0, 0]
        R = 1 + z + z * z / 2 + z ** 3 / 6 + z ** 4 / 24
        assert abs(y - R) <= 4e-16 * max(1.0, abs(R))


def _G(u):  # implicit solution of u' = k u^2 (1 - u):  G(u(t)) - G(u0) = k t
    return math.log(u / (1 - u)) - 1 / u


def test_rk4_order_four_on_nagumo(orc):
    """Error of RK4 with n steps against the exact solution (through G) drops by 2^4 per halving."""
    M = _nag(orc)
    u0, T = 0.3, 0.2
    errs = []
    for n in (4, 8, 16, 32):
        u = orc.rk4(np.array([[u0]]), M, T, n)[0, 0]
        errs.append(abs(_G(u) - _G(u0) - K * T))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(3.8 < r < 4.2 for r in rates), rates


def test_rk4_batch_threads_identical(orc):
    M = _nag(orc)
    u = synth.random_positive_cells(257, 1, 3, lo=0.0, hi=1.0)
    a = orc.rk4(u, M, 5e-3, 2, nthreads=1)
    b = orc.rk4(u, M, 5e-3, 2, nthreads=7)
    assert np.array_equal(a, b)


def test_strang_rk4_reductions(orc):
    """Strang with the RK4 flag: eps = 0 reduces to R_{dt/2} R_{dt/2} leaf by leaf (two RK4 calls of
    T = dt/2, one step each), k = 0 reduces to pure diffusion (Rock4)."""
    dim, J, lmin, eps = 2, 6, 2, 1e-2
    u = front_field(dim, J, 1)
    dt = 1e-2
    g = orc.Grid.build(dim, lmin, J, eps, u.reshape(1, -1))
    _, u0 = g.leaves()
    assert g.strang(_nag(orc), [0.0], dt, orc.STRANG_RK4) == 0
    _, u1 = g.leaves()
    ref = orc.rk4(orc.rk4(u0, _nag(orc), 0.5 * dt, 1), _nag(orc), 0.5 * dt, 1)
    assert np.array_equal(u1, ref)
    g2 = orc.Grid.build(dim, lmin, J, eps, u.reshape(1, -1))
    g3 = orc.Grid.build(dim, lmin, J, eps, u.reshape(1, -1))
    assert g2.strang(_nag(orc, 0.0), [0.1], dt, orc.STRANG_RK4) == 0
    assert g3.diffuse([0.1], dt) is not None
    assert np.array_equal(g2.leaves()[1], g3.leaves()[1])
