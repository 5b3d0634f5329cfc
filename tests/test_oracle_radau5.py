"""Oracle Radau5 (reading O.3) pinned to closed forms, the paper's minimum-
complexity statement and an independent library integrator."""
import numpy as np
import pytest
from scipy.integrate import solve_ivp

import synth


def _R(z):  # Radau IIA stability function, Pade (2,3) approximant of e^z
    return (1 + 2 * z / 5 + z * z / 20) / (1 - 3 * z / 5 + 3 * z * z / 20 - z ** 3 / 60)


def _linear_model(orc, rates):
    """First-order network A_i -> A_j (mass action) = linear ODE y' = M y."""
    reac, prod, rate = [], [], []
    for (i, j, k) in rates:
        reac.append([i, -1])
        prod.append([j, -1])
        rate.append(k)
    m = 1 + max(max(i, j) for i, j, _ in rates)
    spec = dict(kind="mass_action", m=m, reactants=np.array(reac), products=np.array(prod), rate=np.array(rate))
    M = np.zeros((m, m))
    for (i, j, k) in rates:
        M[i, i] -= k
        if j >= 0:
            M[j, i] += k
    return orc.Model(spec), M


def test_stability_function_real(orc):
    """One forced step on y' = lam y reproduces R(h lam) (L-stable: R(-inf) = 0)."""
    model, _ = _linear_model(orc, [(0, -1, 1.0)])
    for z, tol in ((-1.0, 1e-14), (-10.0, 1e-13), (-1e3, 1e-12), (-1e8, 1e-6)):
        y, cnt, st = orc.radau5(np.ones((1, 1)), model, -z, fixed_steps=1)
        assert st[0] == 0
        assert abs(y[0, 0] - _R(z)) <= tol * abs(_R(z))
    assert abs(_R(-1e8)) < 3.1e-8


def test_stability_function_complex(orc):
    """Cyclic first-order network has complex eigenvalues: one forced step must
    equal V R(h Lambda) V^-1 y0 (exercises the complex LU path)."""
    model, M = _linear_model(orc, [(0, 1, 3.0), (1, 2, 5.0), (2, 0, 7.0), (0, -1, 0.5)])
    lam, V = np.linalg.eig(M)
    assert np.abs(lam.imag).max() > 0.5
    y0 = np.array([1.0, 0.2, 0.3])
    for h in (0.05, 0.5, 4.0):
        ref = (V @ np.diag(_R(h * lam)) @ np.linalg.solve(V, y0)).real
        y, _, st = orc.radau5(y0[:, None], model, h, fixed_steps=1)
        assert st[0] == 0
        assert np.allclose(y[:, 0], ref, rtol=1e-12, atol=1e-14)


def test_order_five(orc):
    """Fixed-step convergence on a linear 3x3 system: slope 5 +- 0.3."""
    model, M = _linear_model(orc, [(0, 1, 3.0), (1, 2, 5.0), (2, 0, 7.0), (0, -1, 0.5)])
    from scipy.linalg import expm
    y0 = np.array([1.0, 0.2, 0.3])
    T = 1.0
    ref = expm(M * T) @ y0
    errs = []
    ns = (8, 16, 32)
    for n in ns:
        y, _, _ = orc.radau5(y0[:, None], model, T, fixed_steps=n)
        errs.append(np.abs(y[:, 0] - ref).max())
    slope = np.polyfit(np.log(ns), np.log(errs), 1)[0]
    assert -5.3 < slope < -4.7, (errs, slope)


def test_minimum_complexity_at_equilibrium(orc):
    """minimum complexity = one reaction sub-step and one Newton iteration."""
    model = orc.Model(dict(kind="oregonator"))
    q, fc = 2e-3, 1.6
    b = (-(fc + q - 1) + np.sqrt((fc + q - 1) ** 2 + 4 * q * (fc + 1))) / 2
    y = np.array([[fc * b / (q + b)], [b], [b]])
    _, cnt, st = orc.radau5(y, model, 5e-4)
    c = dict(zip(orc.COUNTER_NAMES, cnt[:, 0]))
    assert st[0] == 0
    assert (c["accept"], c["newton"], c["f"], c["jac"], c["lu"]) == (1, 1, 5, 1, 1)


def _scipy_ref(model, y0, T):
    r = solve_ivp(lambda t, y: model.f(y), (0, T), y0, method="Radau", rtol=1e-13, atol=1e-13,
                  jac=lambda t, y: model.jac(y))
    return r.y[:, -1]


def test_adaptive_accuracy_bz_vs_library(orc):
    """cfg-2 cells over T = 1e-2 at tol 1e-8: normwise error vs scipy Radau (tol 1e-13) <= 1e-7."""
    model = orc.Model(dict(kind="oregonator"))
    u0 = synth.random_bz_cells(6, seed=11)
    u, cnt, st = orc.radau5(u0, model, 1e-2)
    assert (st == 0).all()
    for r in range(u0.shape[1]):
        ref = _scipy_ref(model, u0[:, r], 1e-2)
        assert np.abs(u[:, r] - ref).max() <= 1e-7 * np.abs(ref).max()
    assert cnt[1].min() >= 2  # several accepted steps (stiff transients)


def test_adaptive_accuracy_mass_action_vs_library(orc):
    w = synth.cfg5(J=3)
    model = orc.Model(dict(w.model, m=20))
    u0 = synth.random_positive_cells(2, 20, seed=12)
    u, cnt, st = orc.radau5(u0, model, 5e-5)
    assert (st == 0).all()
    for r in range(2):
        ref = _scipy_ref(model, u0[:, r], 5e-5)
        assert np.abs(u[:, r] - ref).max() <= 1e-7 * np.abs(ref).max()


def test_failure_is_reported(orc):
    """Reading S4: a cell that cannot finish reports failure instead of clipping."""
    model = orc.Model(dict(kind="oregonator"))
    u0 = synth.random_bz_cells(2, seed=13)
    u, cnt, st = orc.radau5(u0, model, 1e-2, max_steps=3)
    assert (st != 0).all()
