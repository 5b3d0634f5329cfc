"""ORACLE (test infrastructure only): Rock4-type coefficient family, regenerated
from the structural definition in PAPER.md §5.3.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
anything under oracle/.  The product never imports this file; it has its own,
independently written generator (paper_1506_04651_b200/tools/gen_rock4.cpp).

PAPER.md P:957-975: Rock4 is "the composition of two methods": a three-term
recurrence of orthogonal polynomials whose length depends on the spectral
radius, and a 4-stage explicit RK finishing formula.  P:976-994: for
dy/dt = Ay the finishing step is a polynomial, evaluated by Horner.  The
ROCK4 tables of the cited Abdulle paper are NOT in PAPER.md; we follow the
reading of SURVEY.md §8(c) O.4 K1 (reading R-K1):

* for s >= 5, n = s - 4, on z in [-l, 0] with x = 1 + 2 z / l, P_n is the
  degree-n polynomial orthogonal for the weight w(z)^2 / sqrt(1 - x^2),
  normalised P_n(0) = 1;
* w(z) = 1 + s1 z + s2 z^2 + s3 z^3 + s4 z^4 is fixed by the order conditions
  R = w P_n = e^z + O(z^5) (sigma from the Taylor coefficients p1..p4 of P_n);
* P_n <-> sigma iterated to a fixed point (damping 1/2, start sigma = 0);
* l_s = largest l (bisection) for which the fixed point converges and
  max_{[-l,0)} |R| <= 1, sampled at max(4e4, 200 s) points uniform on [-l, 0)
  plus 2e4 points uniform on [-min(l, 16), 0), where the interior peak of |R|
  (near z ~ -8, the complex roots of w) lives (DESIGN.md R-K1);
* Gauss-Chebyshev quadrature with 2s+40 nodes; monic recurrence
  pi_{k+1} = (x - a_k) pi_k - b_k pi_{k-1} by the Stieltjes procedure; stage
  coefficients mu_k = (2/l) pi_k(1)/pi_{k+1}(1), nu_k = (1 - a_k) pi_k(1)/pi_{k+1}(1),
  kappa_k = -b_k pi_{k-1}(1)/pi_{k+1}(1).
"""
from __future__ import annotations

import numpy as np


def _stieltjes(xk, wt, n):
    """Monic recurrence coefficients a_k, b_k (k < n) for the discrete measure
    sum_i wt_i delta(x - x_i) (Stieltjes procedure)."""
    a = np.zeros(n)
    b = np.zeros(n)
    p_prev = np.zeros_like(xk)
    p = np.ones_like(xk)
    norm_prev = 1.0
    for k in range(n):
        nk = np.sum(wt * p * p)
        a[k] = np.sum(wt * xk * p * p) / nk
        b[k] = nk / norm_prev if k > 0 else 0.0
        p_next = (xk - a[k]) * p - b[k] * p_prev
        p_prev, p = p, p_next
        norm_prev = nk
    return a, b


def _stage_coeffs(a, b, ell):
    """mu_k, nu_k, kappa_k from the monic recurrence (values at x = 1)."""
    n = len(a)
    pi1 = np.zeros(n + 2)  # pi1[k+1] = pi_k(1), pi1[0] = pi_{-1}(1) = 0
    pi1[1] = 1.0
    for k in range(n):
        pi1[k + 2] = (1.0 - a[k]) * pi1[k + 1] - b[k] * pi1[k]
    mu = np.array([(2.0 / ell) * pi1[k + 1] / pi1[k + 2] for k in range(n)])
    nu = np.array([(1.0 - a[k]) * pi1[k + 1] / pi1[k + 2] for k in range(n)])
    ka = np.array([-b[k] * pi1[k] / pi1[k + 2] for k in range(n)])
    return mu, nu, ka


def taylor_P(mu, nu, ka, order=4):
    """Taylor coefficients of P_n(z) at 0 up to z^order from the normalised recurrence
    P_{k+1} = (nu_k + mu_k z) P_k + kappa_k P_{k-1}, P_0 = 1, P_{-1} = 0."""
    Pm = np.zeros(order + 1)
    P = np.zeros(order + 1)
    P[0] = 1.0
    for k in range(len(mu)):
        zP = np.concatenate([[0.0], P[:-1]])
        Pn = nu[k] * P + mu[k] * zP + ka[k] * Pm
        Pm, P = P, Pn
    return P


def sigma_from_p(p):
    """Order conditions w P = e^z + O(z^5) solved for sigma_1..sigma_4."""
    s1 = 1.0 - p[1]
    s2 = 0.5 - s1 * p[1] - p[2]
    s3 = 1.0 / 6.0 - s2 * p[1] - s1 * p[2] - p[3]
    s4 = 1.0 / 24.0 - s3 * p[1] - s2 * p[2] - s1 * p[3] - p[4]
    return np.array([s1, s2, s3, s4])


def eval_P(mu, nu, ka, z):
    Pm = np.zeros_like(z)
    P = np.ones_like(z)
    for k in range(len(mu)):
        Pn = (nu[k] + mu[k] * z) * P + ka[k] * Pm
        Pm, P = P, Pn
    return P


def eval_w(sig, z):
    return 1.0 + z * (sig[0] + z * (sig[1] + z * (sig[2] + z * sig[3])))


def fixed_point(s, ell, sig0=None, tol=1e-13, maxit=2000):
    """Fixed point P_n <-> sigma for given s, l.  Returns (ok, sigma, mu, nu, kappa)."""
    n = s - 4
    N = 2 * s + 40
    i = np.arange(1, N + 1)
    xk = np.cos((2 * i - 1) * np.pi / (2 * N))  # Gauss-Chebyshev nodes (weights pi/N, constant)
    zk = (xk - 1.0) * ell / 2.0
    sig = np.zeros(4) if sig0 is None else np.array(sig0, dtype=float)
    for _ in range(maxit):
        w = eval_w(sig, zk)
        a, b = _stieltjes(xk, w * w, n)
        mu, nu, ka = _stage_coeffs(a, b, ell)
        new = sigma_from_p(taylor_P(mu, nu, ka))
        nxt = 0.5 * sig + 0.5 * new
        if not np.all(np.isfinite(nxt)):
            return False, sig, None, None, None
        if np.all(np.abs(nxt - sig) <= tol * np.maximum(np.abs(nxt), 1e-300)):
            sig = nxt
            w = eval_w(sig, zk)
            a, b = _stieltjes(xk, w * w, n)
            mu, nu, ka = _stage_coeffs(a, b, ell)
            return True, sig, mu, nu, ka
        sig = nxt
    return False, sig, None, None, None


def n_samples(s):
    return max(40000, 200 * s)


def sample_points(s, ell):
    M = n_samples(s)
    z1 = -ell * np.arange(1, M) / (M - 1)
    zl = min(ell, 16.0)
    z2 = -zl * np.arange(1, 20001) / 20000.0
    return np.concatenate([z1, z2])


def stable(s, ell, sig0=None):
    """Fixed point converged and max |R| <= 1 on [-l, 0).  z = 0 is excluded because
    R(0) = 1 holds exactly in exact arithmetic and its rounding must not decide."""
    ok, sig, mu, nu, ka = fixed_point(s, ell, sig0)
    if not ok:
        return False, sig
    z = sample_points(s, ell)
    R = eval_w(sig, z) * eval_P(mu, nu, ka, z)
    return bool(np.max(np.abs(R)) <= 1.0), sig


def bracket(s):
    """Initial bisection bracket [lo, hi] in units of l; lo stable, hi unstable.
    (The stable set is not an interval over all l > 0 -- for small l the order
    conditions force a huge w -- so the bracket starts near the known l ~ 0.35 s^2
    branch.)"""
    f_lo = 0.2 if s < 7 else (0.25 if s < 12 else 0.28)
    return f_lo * s * s, 0.40 * s * s


def ell_s(s, iters=60):
    """Largest l with a converged fixed point and |R| <= 1 on [-l, 0) (bisection)."""
    lo, hi = bracket(s)
    ok, sig_lo = stable(s, lo)
    assert ok, f"lower bracket unstable for s={s}"
    ok_hi, _ = stable(s, hi, sig_lo)
    assert not ok_hi, f"upper bracket stable for s={s}"
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        ok, sig = stable(s, mid, sig_lo)
        if ok:
            lo, sig_lo = mid, sig
        else:
            hi = mid
        if hi - lo <= 1e-10 * hi:
            break
    return lo


def coefficients(s):
    ell = ell_s(s)
    ok, sig, mu, nu, ka = fixed_point(s, ell)
    assert ok
    return dict(s=s, ell=ell, sigma=sig, mu=mu, nu=nu, kappa=ka)


def write_table(path, s_max=200, workers=8):
    """Text table read by oracle/src (one block per s)."""
    from multiprocessing import Pool
    with Pool(workers) as pool:
        table = pool.map(coefficients, range(5, s_max + 1))
    with open(path, "w") as f:
        f.write("# rock4 oracle table: s ell sigma1..4 then n=s-4 lines mu nu kappa (oracle/rock4_family.py)\n")
        for c in table:
            s = c["s"]
            f.write(f"{s} {c['ell']!r} " + " ".join(repr(float(v)) for v in c["sigma"]) + "\n")
            for k in range(s - 4):
                f.write(f"{float(c['mu'][k])!r} {float(c['nu'][k])!r} {float(c['kappa'][k])!r}\n")


def read_table(path):
    out = {}
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("#")]
    i = 0
    while i < len(lines):
        head = lines[i].split()
        s = int(head[0])
        ell = float(head[1])
        sig = np.array([float(v) for v in head[2:6]])
        rows = np.array([[float(v) for v in lines[i + 1 + k].split()] for k in range(s - 4)])
        out[s] = dict(s=s, ell=ell, sigma=sig, mu=rows[:, 0], nu=rows[:, 1], kappa=rows[:, 2])
        i += 1 + (s - 4)
    return out
