"""Oracle keys (O.1) and models (O.2) against the paper and closed forms."""
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "keys_spec.txt")


def _golden():
    rows = []
    for ln in open(GOLD):
        if ln.startswith("#") or not ln.strip():
            continue
        p = ln.split()
        dim, lev = int(p[0]), int(p[1])
        k = tuple(int(v) for v in p[2:2 + dim])
        rows.append((dim, lev, k, int(p[2 + dim], 2)))
    return rows


def test_keys_golden(orc):
    for dim, lev, k, s in _golden():
        key = orc.key_encode(dim, lev, k)
        assert key == (lev << 58) | s
        assert orc.key_decode(dim, key) == (lev, k)


def test_keys_roundtrip_and_order(orc):
    rng = np.random.default_rng(0)
    for dim, cap in ((2, 29), (3, 19)):
        for _ in range(300):
            lev = int(rng.integers(0, cap + 1))
            k = tuple(int(x) for x in rng.integers(0, 1 << lev, size=dim)) if lev else (0,) * dim
            assert orc.key_decode(dim, orc.key_encode(dim, lev, k)) == (lev, k)
    # children of a node are consecutive keys in Morton child order
    p = orc.key_encode(2, 1, (1, 0))
    ch = [orc.key_encode(2, 2, (2 + bx, 0 + by)) for bx in (0, 1) for by in (0, 1)]
    assert ch == sorted(ch) and [c & 0xF for c in ch] == [0b1000, 0b1001, 0b1010, 0b1011]
    assert (ch[0] & ((1 << 58) - 1)) >> 2 == p & ((1 << 58) - 1)


def _fd_jac(model, u, h=1e-7):
    m = len(u)
    J = np.zeros((m, m))
    for j in range(m):
        e = np.zeros(m)
        e[j] = h * max(1.0, abs(u[j]))
        J[:, j] = (model.f(u + e) - model.f(u - e)) / (2 * e[j])
    return J


def test_oregonator_paper_form(orc):
    """PAPER.md P:271-275 prints the BZ RHS with q = 0.02, 1/mu = 1e5, 1/eps = 1e2;
    the generic Oregonator with q = 0.02 must equal it."""
    M = orc.Model(dict(kind="oregonator", q=0.02))
    rng = np.random.default_rng(1)
    for _ in range(50):
        u1, u2, u3 = rng.uniform(0, 2, 3)
        paper = np.array([1e5 * (-0.02 * u1 - u2 * u1 + 1.6 * u3),
                          1e2 * (u2 - u2 ** 2 - u1 * (u2 - 0.02)),
                          u2 - u3])
        assert np.allclose(M.f([u1, u2, u3]), paper, rtol=1e-13, atol=1e-9)


def test_oregonator_steady_state_and_jacobian(orc):
    M = orc.Model(dict(kind="oregonator"))
    q, fc = 2e-3, 1.6
    b = (-(fc + q - 1) + np.sqrt((fc + q - 1) ** 2 + 4 * q * (fc + 1))) / 2
    y = np.array([fc * b / (q + b), b, b])
    assert np.allclose(y, [1.29574132, 0.00851737, 0.00851737], atol=1e-8)
    assert np.max(np.abs(M.f(y))) < 1e-9
    assert np.array_equal(M.f(np.zeros(3)), np.zeros(3))
    rng = np.random.default_rng(2)
    mx = 0.0
    for _ in range(100):
        bb, cc = rng.uniform(0, 1, 2)
        u = np.array([fc * cc / (q + bb), bb, cc])
        J = M.jac(u)
        assert np.allclose(J, _fd_jac(M, u), rtol=1e-6, atol=1e-6 * np.abs(J).max())
        mx = max(mx, np.abs(np.linalg.eigvals(J)).max())
    # Jacobian eigenvalue amplitude "of the order of 10^5"
    assert 2e4 < mx < 5e5


def test_mass_action_properties(orc):
    w = synth.cfg5(J=3)
    M = orc.Model(dict(w.model, m=20))
    rng = np.random.default_rng(3)
    for _ in range(20):
        u = rng.uniform(0.01, 1.0, 20)
        J = M.jac(u)
        assert np.allclose(J, _fd_jac(M, u), rtol=1e-5, atol=1e-6 * np.abs(J).max())
        assert M.f(u).sum() <= 1e-9 * np.abs(M.f(u)).sum()  # species count non-increasing
        z = u.copy()
        i = int(rng.integers(20))
        z[i] = 0.0
        assert M.f(z)[i] >= 0.0  # positivity
