"""ORACLE — test infrastructure only.

ctypes binding of oracle/liboracle.so (plain scalar C++ in oracle/src, built
with -O2 -ffp-contract=off) plus the oracle's Rock4 coefficient table
(oracle/rock4_family.py -> oracle/data/rock4_oracle.txt).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package.  It shares no code with paper_1506_04651_b200/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = [os.path.join(HERE, "src", f) for f in ("core.cpp", "mr.cpp", "capi.cpp")]
TABLE = os.path.join(HERE, "data", "rock4_oracle.txt")

_lib = None


def build(force: bool = False) -> str:
    deps = SRC + [os.path.join(HERE, "src", "oracle.hpp")]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(p) for p in deps):
        return LIB
    cmd = ["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", LIB] + SRC
    subprocess.check_call(cmd)
    return LIB


class _Model(C.Structure):
    _fields_ = [("kind", C.c_int), ("m", C.c_int), ("q", C.c_double), ("f_c", C.c_double),
                ("eps_b", C.c_double), ("mu", C.c_double), ("n_reac", C.c_int),
                ("reactants", C.c_void_p), ("products", C.c_void_p), ("rate", C.c_void_p), ("k_nag", C.c_double)]


class _R5(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("h0", C.c_double), ("nit", C.c_int),
                ("max_steps", C.c_int64), ("fixed_steps", C.c_int)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp, dp, i64, i32p = C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int32)
        L.or_key_encode.restype = C.c_uint64
        L.or_key_encode.argtypes = [C.c_int, C.c_int, i32p]
        L.or_key_decode.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_int), i32p]
        L.or_model_f.argtypes = [C.POINTER(_Model), dp, dp]
        L.or_model_jac.argtypes = [C.POINTER(_Model), dp, dp]
        L.or_grid_set_operator.argtypes = [vp, C.c_int]
        L.or_grid_set_operator.restype = None
        L.or_rk4_batch.argtypes = [i64, C.POINTER(_Model), dp, C.c_double, C.c_int, C.c_int]
        L.or_radau5_batch.argtypes = [i64, C.POINTER(_Model), dp, C.c_double, C.POINTER(_R5), C.c_int,
                                      C.POINTER(C.c_int64), i32p]
        L.or_rock4_load.argtypes = [C.c_char_p]
        L.or_rock4_get.argtypes = [C.c_int, dp, dp, dp, dp, dp]
        L.or_grid_build.restype = vp
        L.or_grid_build.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, dp, C.POINTER(C.c_int)]
        L.or_grid_from_leaves.restype = vp
        L.or_grid_from_leaves.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, i64,
                                          C.POINTER(C.c_uint64), dp, C.POINTER(C.c_int)]
        L.or_grid_free.argtypes = [vp]
        L.or_grid_nleaves.restype = i64
        L.or_grid_nleaves.argtypes = [vp]
        L.or_grid_nnodes.restype = i64
        L.or_grid_nnodes.argtypes = [vp]
        L.or_grid_leaves.argtypes = [vp, C.POINTER(C.c_uint64), dp]
        L.or_grid_set_values.argtypes = [vp, dp]
        L.or_grid_adapt.argtypes = [vp]
        L.or_threshold_sq.restype = C.c_double
        L.or_threshold_sq.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int]
        L.or_predict_vals.restype = C.c_double
        L.or_predict_vals.argtypes = [C.c_int, dp, C.POINTER(C.c_int)]
        L.or_grid_check.argtypes = [vp]
        L.or_grid_rho1.restype = C.c_double
        L.or_grid_rho1.argtypes = [vp]
        L.or_grid_apply.argtypes = [vp, dp, dp]
        L.or_grid_rock4_species.argtypes = [vp, dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                            C.POINTER(C.c_int64)]
        L.or_grid_rock4_forced.argtypes = [vp, dp, C.c_double, C.c_double, C.c_int, dp, dp]
        L.or_grid_diffuse.argtypes = [vp, dp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                      C.POINTER(C.c_int64)]
        L.or_grid_react.argtypes = [vp, C.POINTER(_Model), C.c_double, C.POINTER(_R5), C.c_int,
                                    C.POINTER(C.c_int64)]
        L.or_strang_step.argtypes = [vp, C.POINTER(_Model), dp, C.c_double, C.c_int, C.POINTER(_R5),
                                     C.c_double, C.c_double, C.c_int, C.c_int]
        smax = L.or_rock4_load(TABLE.encode())
        if smax < 5:
            raise RuntimeError(f"oracle Rock4 table missing or invalid: {TABLE}")
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Model:
    """Holds the ctypes struct and keeps the arrays alive."""

    def __init__(self, spec: dict, m: int = 3):
        kind = spec.get("kind", "oregonator")
        self.s = _Model()
        if kind == "oregonator":
            self.s.kind, self.s.m = 1, 3
            self.s.q, self.s.f_c = spec.get("q", 2e-3), spec.get("f_c", 1.6)
            self.s.eps_b, self.s.mu = spec.get("eps_b", 1e-2), spec.get("mu", 1e-5)
        elif kind == "nagumo":  # m = 1, f = k u^2 (1 - u)
            self.s.kind, self.s.m = 3, 1
            self.s.k_nag = spec.get("k", 10.0)
        else:
            self.reac = np.ascontiguousarray(spec["reactants"], dtype=np.int32)
            self.prod = np.ascontiguousarray(spec["products"], dtype=np.int32)
            self.rate = np.ascontiguousarray(spec["rate"], dtype=np.float64)
            self.s.kind, self.s.m = 2, int(spec.get("m", m))
            self.s.n_reac = len(self.rate)
            self.s.reactants = self.reac.ctypes.data
            self.s.products = self.prod.ctypes.data
            self.s.rate = self.rate.ctypes.data
        self.m = self.s.m

    def f(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(self.m)
        lib().or_model_f(C.byref(self.s), _dp(u), _dp(out))
        return out

    def jac(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros((self.m, self.m))
        lib().or_model_jac(C.byref(self.s), _dp(u), _dp(out))
        return out


def r5opts(rtol=1e-8, atol=1e-8, h0=0.0, nit=7, max_steps=100000, fixed_steps=0):
    o = _R5()
    o.rtol, o.atol, o.h0, o.nit, o.max_steps, o.fixed_steps = rtol, atol, h0, nit, max_steps, fixed_steps
    return o


def radau5(u, model: Model, T, nthreads=1, **opts):
    """Integrate each column of u[m, n] over [0, T].  Returns (u_out, counters[7, n], status[n])."""
    u = np.array(u, dtype=np.float64, order="C", copy=True)
    m, n = u.shape
    assert m == model.m
    cnt = np.zeros((7, n), dtype=np.int64)
    st = np.zeros(n, dtype=np.int32)
    o = r5opts(**opts)
    lib().or_radau5_batch(n, C.byref(model.s), _dp(u), T, C.byref(o), nthreads,
                          cnt.ctypes.data_as(C.POINTER(C.c_int64)), st.ctypes.data_as(C.POINTER(C.c_int32)))
    return u, cnt, st


def rk4(u, model: Model, T, nsteps=1, nthreads=1):
    """Classical RK4 on each column of u[m, n] over [0, T] in nsteps equal steps (A10)."""
    u = np.array(u, dtype=np.float64, order="C", copy=True)
    m, n = u.shape
    assert m == model.m
    lib().or_rk4_batch(n, C.byref(model.s), _dp(u), T, int(nsteps), nthreads)
    return u


STRANG_RK4 = 0x100  # Strang scheme flag: reaction by RK4 with h_max = opts h0 (reading R-K4)

COUNTER_NAMES = ("attempt", "accept", "reject", "f", "jac", "lu", "newton")


def key_encode(dim, level, k):
    kk = (C.c_int32 * 3)(*(list(k) + [0] * (3 - len(k))))
    return int(lib().or_key_encode(dim, level, kk))


def key_decode(dim, key):
    lv = C.c_int()
    kk = (C.c_int32 * 3)()
    lib().or_key_decode(dim, C.c_uint64(key), C.byref(lv), kk)
    return lv.value, tuple(kk[:dim])


def threshold_sq(dim, lmax, eps, j):
    """The oracle's E_j = eps_j^2 = eps^2 2^{d(j-J)}, compared with Q on both sides."""
    return float(lib().or_threshold_sq(dim, lmax, eps, j))


def predict_vals(dim, v, cb):
    """The oracle's tensor-product prediction (Eq. inter_1d) of the child with bits cb
    from the 3^d parent-level values v (index (oz*3+oy)*3+ox)."""
    v = np.ascontiguousarray(v, dtype=np.float64).ravel()
    assert v.size == 3 ** dim
    c = (C.c_int * 3)(*(list(cb) + [0] * (3 - len(cb))))
    return float(lib().or_predict_vals(dim, _dp(v), c))


def rock4_coeffs(s):
    ell = C.c_double()
    sig = np.zeros(4)
    mu, nu, ka = np.zeros(s - 4), np.zeros(s - 4), np.zeros(s - 4)
    if lib().or_rock4_get(s, C.byref(ell), _dp(sig), _dp(mu), _dp(nu), _dp(ka)) != 0:
        raise ValueError(s)
    return dict(s=s, ell=ell.value, sigma=sig, mu=mu, nu=nu, kappa=ka)


class Grid:
    """Oracle MR grid (hash map over all tree nodes)."""

    def __init__(self, ptr, dim, m):
        self.p, self.dim, self.m = ptr, dim, m

    @classmethod
    def build(cls, dim, lmin, lmax, eps, u_rowmajor):
        u = np.ascontiguousarray(u_rowmajor, dtype=np.float64)
        m = u.shape[0]
        rc = C.c_int()
        p = lib().or_grid_build(dim, lmin, lmax, eps, m, _dp(u), C.byref(rc))
        g = cls(p, dim, m)
        if rc.value != 0:
            raise RuntimeError(f"oracle grid_build rc={rc.value}")
        return g

    @classmethod
    def from_leaves(cls, dim, lmin, lmax, eps, keys, u):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        rc = C.c_int()
        p = lib().or_grid_from_leaves(dim, lmin, lmax, eps, u.shape[0], len(keys),
                                      keys.ctypes.data_as(C.POINTER(C.c_uint64)), _dp(u), C.byref(rc))
        g = cls(p, dim, u.shape[0])
        if rc.value != 0:
            raise RuntimeError(f"oracle grid_from_leaves rc={rc.value}")
        return g

    def __del__(self):
        if getattr(self, "p", None):
            lib().or_grid_free(self.p)
            self.p = None

    @property
    def n_leaves(self):
        return int(lib().or_grid_nleaves(self.p))

    @property
    def n_nodes(self):
        return int(lib().or_grid_nnodes(self.p))

    def leaves(self):
        n = self.n_leaves
        keys = np.zeros(n, dtype=np.uint64)
        u = np.zeros((self.m, n))
        lib().or_grid_leaves(self.p, keys.ctypes.data_as(C.POINTER(C.c_uint64)), _dp(u))
        return keys, u

    def set_values(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        assert u.shape == (self.m, self.n_leaves)
        lib().or_grid_set_values(self.p, _dp(u))

    def adapt(self):
        rc = lib().or_grid_adapt(self.p)
        if rc != 0:
            raise RuntimeError(f"oracle adapt rc={rc}")

    def check(self):
        return lib().or_grid_check(self.p)

    def set_operator(self, mode):
        """0 = ghost values by MR prediction (default), 1 = two-point fluxes (N4, reading R-T)."""
        lib().or_grid_set_operator(self.p, int(mode))

    @property
    def rho1(self):
        return float(lib().or_grid_rho1(self.p))

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        lib().or_grid_apply(self.p, _dp(x), _dp(y))
        return y

    def rock4(self, x, eps_i, T, rtol=1e-8, atol=1e-8, s_max=200):
        x = np.array(x, dtype=np.float64, copy=True)
        st = np.zeros(5, dtype=np.int64)
        rc = lib().or_grid_rock4_species(self.p, _dp(x), eps_i, T, rtol, atol, s_max,
                                         st.ctypes.data_as(C.POINTER(C.c_int64)))
        if rc != 0:
            raise RuntimeError(f"oracle rock4 rc={rc}")
        return x, dict(zip(("steps", "rejects", "matvecs", "s_min", "s_max"), st.tolist()))

    def rock4_forced(self, x, eps_i, h, s):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out, e = np.zeros_like(x), np.zeros_like(x)
        if lib().or_grid_rock4_forced(self.p, _dp(x), eps_i, h, s, _dp(out), _dp(e)) != 0:
            raise ValueError(s)
        return out, e

    def diffuse(self, eps_diff, T, rtol=1e-8, atol=1e-8, s_max=200, nthreads=8):
        eps = np.ascontiguousarray(eps_diff, dtype=np.float64)
        st = np.zeros(5, dtype=np.int64)
        rc = lib().or_grid_diffuse(self.p, _dp(eps), T, rtol, atol, s_max, nthreads,
                                   st.ctypes.data_as(C.POINTER(C.c_int64)))
        if rc != 0:
            raise RuntimeError(f"oracle diffuse rc={rc}")
        return dict(zip(("steps", "rejects", "matvecs", "s_min", "s_max"), st.tolist()))

    def react(self, model: Model, T, nthreads=8, **opts):
        nf = C.c_int64()
        o = r5opts(**opts)
        lib().or_grid_react(self.p, C.byref(model.s), T, C.byref(o), nthreads, C.byref(nf))
        return int(nf.value)

    def strang(self, model: Model, eps_diff, dt, scheme=0, nthreads=8, krtol=1e-8, katol=1e-8, ks_max=200,
               **opts):
        eps = np.ascontiguousarray(eps_diff, dtype=np.float64)
        o = r5opts(**opts)
        return lib().or_strang_step(self.p, C.byref(model.s), _dp(eps), dt, scheme, C.byref(o), krtol, katol,
                                    ks_max, nthreads)
