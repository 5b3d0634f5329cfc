"""CPU-side checks of the product boundary: librdmr.so loads, exports every symbol include/rdmr.h
declares, and its pure host helpers (keys, status strings, Rock4 table) behave.  No compute calls."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "rdmr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:rd|mr)_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def P():
    from paper_1506_04651_b200 import build
    build.build()
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def test_every_declared_symbol_exported(P):
    names = _declared()
    assert len(names) >= 16
    L = P.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(P.SYMBOLS)


def test_no_cpu_fallback_in_binding():
    src = open(os.path.join(ROOT, "paper_1506_04651_b200", "__init__.py")).read()
    assert "import oracle" not in src and "from oracle" not in src
    for f in os.listdir(os.path.join(ROOT, "paper_1506_04651_b200", "csrc")):
        txt = open(os.path.join(ROOT, "paper_1506_04651_b200", "csrc", f)).read()
        assert not re.search(r'#include\s*["<][^">]*oracle', txt), f


def test_status_strings(P):
    assert P.status_string(0) == "ok"
    assert "Radau5" in P.status_string(P.RD_ESTIFF)
    assert P.status_string(123) == "unknown status"


def test_keys_match_paper_examples(P, orc):
    """P:749-753 interleaving (x first); SPEC examples via tests/golden/keys_spec.txt (also pin the oracle)."""
    rng = np.random.default_rng(0)
    for dim in (2, 3):
        for _ in range(300):
            j = int(rng.integers(0, 14 if dim == 2 else 9))
            k = [int(rng.integers(0, 1 << j)) if j else 0 for _ in range(dim)]
            key = P.mr_key_encode(dim, j, k)
            assert key == orc.key_encode(dim, j, k)
            assert P.mr_key_decode(dim, key) == (j, tuple(k))
    # d=2, level 2, k=(2,1): digits x1 y1 x2 y2 = 1 0 0 1 -> s = 1001b = 9
    assert P.mr_key_encode(2, 2, (2, 1)) == (2 << 58) | 0b1001


def test_rock4_table_properties(P):
    """Library table (paper_1506_04651_b200/tools/gen_rock4.cpp): order conditions R = e^z + O(z^5),
    |R_s| <= 1 on [-ell_s, 0], nu + kappa = 1, ell_s / s^2 -> ~0.35 ("grows like s^2")."""
    smax = P.rock4_smax()
    assert smax >= 40
    for s in list(range(5, 13)) + [smax // 2, smax]:
        c = P.rock4_coeffs(s)
        assert np.allclose(c["nu"] + c["kappa"], 1.0, atol=1e-12)
        z = -np.linspace(0, c["ell"], 20001)[1:]
        Pm, Pc = np.zeros_like(z), np.ones_like(z)
        for mu, nu, ka in zip(c["mu"], c["nu"], c["kappa"]):
            Pm, Pc = Pc, (nu + mu * z) * Pc + ka * Pm
        sg = c["sigma"]
        R = (1 + z * (sg[0] + z * (sg[1] + z * (sg[2] + z * sg[3])))) * Pc
        # the interior peak (z ~ -8) sits ON the boundary |R| = 1 by construction of ell_s (R-K1);
        # re-evaluating the double-rounded table in double lands within 1e-5 of it
        assert np.abs(R).max() <= 1 + 1e-5
        # order 4: R(z) - e^z = O(z^5) near 0
        for zz in (-1e-2, -2e-2):
            Pm, Pc = 0.0, 1.0
            for mu, nu, ka in zip(c["mu"], c["nu"], c["kappa"]):
                Pm, Pc = Pc, (nu + mu * zz) * Pc + ka * Pm
            Rz = (1 + zz * (sg[0] + zz * (sg[1] + zz * (sg[2] + zz * sg[3])))) * Pc
            assert abs(Rz - np.exp(zz)) <= 5 * abs(zz) ** 5
    assert 0.33 <= P.rock4_coeffs(smax)["ell"] / smax ** 2 <= 0.37


def test_rock4_table_vs_oracle(P, orc):
    """Two independent generators of the same family (R-K1).  ell_s sits where an interior peak of
    |R| touches 1, so the two stability tests (double, sampled vs long double, peak-refined) place it
    within ~1e-5; at the SAME ell the two fixed points (Stieltjes/numpy vs Lanczos/long double)
    must agree to rounding."""
    from oracle import rock4_family as F
    for s in (5, 6, 9, 17, 33, 64, 120, 200):
        if s > P.rock4_smax():
            continue
        a, b = P.rock4_coeffs(s), orc.rock4_coeffs(s)
        assert a["ell"] == pytest.approx(b["ell"], rel=1e-4)
        ok, sig, mu, nu, ka = F.fixed_point(s, a["ell"])
        assert ok
        assert np.allclose(a["sigma"], sig, rtol=1e-9, atol=1e-14)
        assert np.allclose(a["mu"], mu, rtol=1e-9, atol=1e-16)
        assert np.allclose(a["nu"], nu, rtol=1e-9, atol=1e-14)
        assert np.allclose(a["kappa"], ka, rtol=1e-8, atol=1e-14)
