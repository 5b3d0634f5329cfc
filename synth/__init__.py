"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module is shared by the oracle side (``oracle/``) and the product side
(``paper_1506_04651_b200``).  It holds NO arithmetic of the method (no
Radau5, Rock4, multiresolution, Morton keys or FV operator): it only draws
random numbers with splitmix64 and evaluates the initial-condition recipes of
SURVEY.md §8(d) at level-J cell centres.  Grids are returned ROW-MAJOR with
axis 1 (x, Morton-most-significant coordinate) fastest, i.e. numpy shape
``[m, ny, nx]`` (2-D) or ``[m, nz, ny, nx]`` (3-D).  Each side converts to its
own layout with its own code.

PAPER.md never prints its initial data (SPEC.md S:619 agrees); the recipes
here are the DESIGN.md input recipe, shaped like the paper's workloads
(BZ fronts; STROKE-like stiff m~20 chemistry).

Random numbers: splitmix64 (Steele, Lea, Flood 2014), doubles as
``(x >> 11) * 2**-53``, seed = configuration index (1..5).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


class SplitMix64:
    """Sequential splitmix64 stream (scalar draws, exact integer arithmetic)."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + _GAMMA) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * _M1) & _MASK
        z = ((z ^ (z >> 27)) * _M2) & _MASK
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)
        return lo + (hi - lo) * u

    def uniform_block(self, n: int) -> np.ndarray:
        """n consecutive draws U[0,1) (vectorised; identical to n scalar draws)."""
        i = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + i * np.uint64(_GAMMA)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * _GAMMA) & _MASK
        return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# ---------------------------------------------------------------- BZ model
OREGONATOR = dict(q=2e-3, f_c=1.6, eps_b=1e-2, mu=1e-5)  # BJ configs[0]; SURVEY C1
BZ_EPS_DIFF = (2.5e-3, 2.5e-3, 1.5e-3)


def _S(t):
    return 0.5 * (1.0 + np.tanh(t))


def _centres(n: int, dim: int):
    x = (np.arange(n, dtype=np.float64) + 0.5) / n
    if dim == 2:
        yy, xx = np.meshgrid(x, x, indexing="ij")
        return xx, yy
    zz, yy, xx = np.meshgrid(x, x, x, indexing="ij")
    return xx, yy, zz


def _bz_state(b, c, q=OREGONATOR["q"], f_c=OREGONATOR["f_c"]):
    a = f_c * c / (q + b)  # quasi-steady a (BJ configs[0]: "a at its quasi-steady value")
    return np.stack([a, b, c])


@dataclass
class Workload:
    name: str
    dim: int              # 0 = independent cells (cfg 2)
    level_max: int        # J
    level_min: int        # L_min
    eps_mr: float
    m: int
    u: np.ndarray         # row-major [m, (nz,) ny, nx] or [m, n] for cfg 2
    eps_diff: tuple
    dt: float
    steps: int
    model: dict = field(default_factory=dict)


def cfg1(J: int = 7) -> Workload:
    """BJ configs[0]: 2-D uniform 128^2 BZ, K=4 circular fronts (SURVEY §8(d) cfg 1)."""
    rng = SplitMix64(1)
    fronts = []
    for _ in range(4):
        cx = rng.uniform(0.15, 0.85)
        cy = rng.uniform(0.15, 0.85)
        r = rng.uniform(0.08, 0.2)
        fronts.append((cx, cy, r))
    n = 1 << J
    xx, yy = _centres(n, 2)
    delta = 2.0 / 128.0
    phi = np.zeros_like(xx)
    phi2 = np.zeros_like(xx)
    for cx, cy, r in fronts:
        dist = np.hypot(xx - cx, yy - cy)
        phi = np.maximum(phi, _S((r - dist) / delta))
        phi2 = np.maximum(phi2, _S((r - 0.03 - dist) / delta))
    b = 0.05 + 0.75 * phi
    c = 0.05 + 0.45 * phi2
    return Workload("cfg1", 2, J, J, 0.0, 3, _bz_state(b, c), BZ_EPS_DIFF, 1e-3, 1,
                    dict(kind="oregonator", **OREGONATOR))


def cfg2(n: int = 1 << 22) -> Workload:
    """BJ configs[1]: independent BZ cells, (b,c) ~ U[0,1)^2, a quasi-steady."""
    rng = SplitMix64(2)
    d = rng.uniform_block(2 * n).reshape(n, 2)
    b, c = d[:, 0].copy(), d[:, 1].copy()
    return Workload("cfg2", 0, 0, 0, 0.0, 3, _bz_state(b, c), BZ_EPS_DIFF, 1e-2, 1,
                    dict(kind="oregonator", **OREGONATOR))


def _spiral_draws(rng: SplitMix64, K: int, twist: bool):
    cores = []
    for _ in range(K):
        cx = rng.uniform(0.1, 0.9)
        cy = rng.uniform(0.1, 0.9)
        ph0 = rng.uniform(0.0, 2.0 * math.pi)
        lam = rng.uniform(0.08, 0.15)
        R = rng.uniform(0.1, 0.2)
        tau = rng.uniform(0.5, 1.5) if twist else 0.0
        cores.append((cx, cy, ph0, lam, R, tau))
    return cores


def _spiral_fields(coords, cores, delta):
    xx, yy = coords[0], coords[1]
    zz = coords[2] if len(coords) == 3 else None
    A = np.zeros_like(xx)
    C = np.zeros_like(xx)
    for cx, cy, ph0, lam, R, tau in cores:
        dx, dy = xx - cx, yy - cy
        r = np.hypot(dx, dy)
        th = np.arctan2(dy, dx)
        ph = th - ph0 - 2.0 * math.pi * r / lam
        if zz is not None:
            ph = ph - 2.0 * math.pi * tau * zz
        env = _S((R - r) / delta)
        A = np.maximum(A, _S((np.cos(ph) - 0.8) / 0.05) * env)
        C = np.maximum(C, _S((np.cos(ph + 0.6) - 0.8) / 0.05) * env)
    return A, C


def cfg3(J: int = 10, K: int = 6) -> Workload:
    """BJ configs[2]: 2-D MR J=10, L_min=4, eps=1e-2, spiral-like fronts (K=6, seed 3)."""
    rng = SplitMix64(3)
    cores = _spiral_draws(rng, K, twist=False)
    n = 1 << J
    A, C = _spiral_fields(_centres(n, 2), cores, 3.0 / 1024.0)
    b = 0.05 + 0.75 * A
    c = 0.05 + 0.4 * C
    return Workload("cfg3", 2, J, 4, 1e-2, 3, _bz_state(b, c), BZ_EPS_DIFF, 1e-3, 20,
                    dict(kind="oregonator", **OREGONATOR))


def cfg4(J: int = 7, K: int = 8) -> Workload:
    """BJ configs[3]: 3-D MR J=7, L_min=3, eps=1e-2, twisted scroll waves (K=8, seed 4)."""
    rng = SplitMix64(4)
    cores = _spiral_draws(rng, K, twist=True)
    n = 1 << J
    A, C = _spiral_fields(_centres(n, 3), cores, 3.0 / 128.0)
    b = 0.05 + 0.75 * A
    c = 0.05 + 0.4 * C
    return Workload("cfg4", 3, J, 3, 1e-2, 3, _bz_state(b, c), BZ_EPS_DIFF, 1e-3, 10,
                    dict(kind="oregonator", **OREGONATOR))


def mass_action_network(rng: SplitMix64, m: int = 20, n_reac: int = 40):
    """Synthetic mass-action network (SURVEY §8(d) cfg 5 draw order)."""
    reactants = -np.ones((n_reac, 2), dtype=np.int32)
    products = -np.ones((n_reac, 2), dtype=np.int32)
    rate = np.zeros(n_reac)
    for r in range(n_reac):
        order = 1 + (1 if rng.uniform() < 0.5 else 0)
        for s in range(order):
            reactants[r, s] = int(math.floor(m * rng.uniform()))
        nprod = 1 if order == 1 else 1 + (1 if rng.uniform() < 0.5 else 0)
        reac_set = set(int(v) for v in reactants[r] if v >= 0)
        for s in range(nprod):
            while True:
                p = int(math.floor(m * rng.uniform()))
                if p not in reac_set:
                    break
            products[r, s] = p
        rate[r] = 10.0 ** (-2.0 + 8.0 * rng.uniform())
    return reactants, products, rate


def cfg5(J: int = 9, m: int = 20) -> Workload:
    """BJ configs[4]: 2-D uniform 512^2, m=20 mass-action network, 5 steps dt=1e-4."""
    rng = SplitMix64(5)
    reactants, products, rate = mass_action_network(rng, m, 40)
    eps = tuple(1e-4 + (5e-3 - 1e-4) * rng.uniform() for _ in range(m))
    n = 1 << J
    xx, yy = _centres(n, 2)
    u = np.empty((m, n, n))
    for i in range(m):
        ci = 0.1 + 0.9 * rng.uniform()
        ni = 1 + int(math.floor(3 * rng.uniform()))
        pi_ = 1 + int(math.floor(3 * rng.uniform()))
        phi = rng.uniform()
        psi = rng.uniform()
        u[i] = ci * (1.0 + 0.5 * np.cos(2 * math.pi * (ni * xx + phi)) * np.cos(2 * math.pi * (pi_ * yy + psi)))
    return Workload("cfg5", 2, J, J, 0.0, m, u, eps, 1e-4, 5,
                    dict(kind="mass_action", reactants=reactants, products=products, rate=rate))


NAGUMO = dict(k=10.0)        # f = k u^2 (1 - u), k = 10
NAGUMO_EPS_DIFF = (0.1,)     # eps_1 = 0.1


def cfg6(J: int = 10, K: int = 8) -> Workload:
    """SURVEY §8(f) N1 (not a BJ config): NAGUMO (m = 1) on a 2-D MR grid J=10, L_min=4, eps=1e-2, dt=1e-2
    (P:259-268); 0 <= u0 <= 1: K seeded discs u = max_k S((r_k - |x - c_k|)/delta), delta = 0.003,
    draws per disc in order c_k ~ U[0.2,0.8]^2 (x then y), r_k ~ U[0.05,0.15], seed 6.  The fronts then
    travel as NAGUMO waves."""
    rng = SplitMix64(6)
    discs = []
    for _ in range(K):
        cx = rng.uniform(0.2, 0.8)
        cy = rng.uniform(0.2, 0.8)
        r = rng.uniform(0.05, 0.15)
        discs.append((cx, cy, r))
    n = 1 << J
    xx, yy = _centres(n, 2)
    u = np.zeros_like(xx)
    for cx, cy, r in discs:
        u = np.maximum(u, _S((r - np.hypot(xx - cx, yy - cy)) / 0.003))
    return Workload("cfg6", 2, J, 4, 1e-2, 1, u[None], NAGUMO_EPS_DIFF, 1e-2, 20, dict(kind="nagumo", **NAGUMO))


CONFIGS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5, 6: cfg6}


def random_bz_cells(n: int, seed: int) -> np.ndarray:
    """Extra seeded BZ cells (same recipe as cfg 2, other seed) for parity cases."""
    rng = SplitMix64(seed)
    d = rng.uniform_block(2 * n).reshape(n, 2)
    return _bz_state(d[:, 0].copy(), d[:, 1].copy())


def random_positive_cells(n: int, m: int, seed: int, lo=0.05, hi=1.0) -> np.ndarray:
    """Seeded positive concentrations [m, n] for mass-action parity cases."""
    rng = SplitMix64(seed)
    return lo + (hi - lo) * rng.uniform_block(n * m).reshape(m, n)
