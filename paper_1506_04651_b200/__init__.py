"""Thin ctypes binding of librdmr.so (include/rdmr.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of librdmr.so; this module converts torch
CUDA tensors to raw device pointers and the current stream to a cudaStream_t, and raises on a
non-OK status.  There is no CPU fallback: without the built library or a CUDA device every call
raises.  Names follow the C-ABI (and the paper's notation).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RDMR_LIB") or os.path.join(HERE, "librdmr.so")

RD_OK, RD_EINVAL, RD_ENOMEM, RD_ECUDA, RD_ESTIFF, RD_ESTRUCT, RD_ENOTSUP = 0, -1, -2, -3, -4, -5, -6
RD_MODEL_OREGONATOR, RD_MODEL_MASS_ACTION, RD_MODEL_NAGUMO = 1, 2, 3
RD_STRANG_RDR, RD_STRANG_DRD = 0, 1
RD_STRANG_RK4 = 0x100  # scheme flag: RK4 reaction substeps (h_max = radau5 opts h0)
RD_OP_PREDICTION, RD_OP_TWO_POINT, RD_OP_TWO_POINT_COMPACT = 0, 1, 2  # mr_set_operator modes
COUNTER_NAMES = ("attempt", "accept", "reject", "f", "jac", "lu", "newton", "status")

# every symbol include/rdmr.h declares (checked by tests/test_abi.py)
SYMBOLS = ("rd_status_string", "mr_grid_build", "mr_adapt", "mr_grid_leaves", "mr_grid_info", "mr_grid_free",
           "mr_key_encode", "mr_key_decode", "mr_rowmajor_to_morton", "rd_fv_apply", "rd_reaction_radau5",
           "rd_diffusion_rock4", "rd_rock4_forced_step", "rd_strang_step", "rd_rock4_smax", "rd_rock4_coeffs",
           "rd_kernel_launches", "mr_grid_stats", "rd_reaction_rk4", "mr_set_operator",
           "rd_reaction_radau5_cells", "rd_reaction_cost", "rd_shard_bounds")


class RdError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        super().__init__(f"{fn}: {status_string(status)} ({status})")


class mr_params(C.Structure):
    _fields_ = [("dim", C.c_int), ("level_min", C.c_int), ("level_max", C.c_int), ("eps_mr", C.c_double)]


class rd_model(C.Structure):
    _fields_ = [("kind", C.c_int), ("m", C.c_int), ("q", C.c_double), ("f_c", C.c_double),
                ("eps_b", C.c_double), ("mu", C.c_double), ("n_reac", C.c_int),
                ("reactants", C.c_void_p), ("products", C.c_void_p), ("rate", C.c_void_p), ("k_nag", C.c_double)]


class rd_radau5_opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("h0", C.c_double), ("nit", C.c_int),
                ("max_steps", C.c_int64)]


class rd_rock4_opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("s_max", C.c_int)]


class rd_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_cells", "n_attempts", "n_accept", "n_reject", "n_f", "n_jac", "n_lu",
                                         "n_newton", "n_failed", "rock4_steps", "rock4_rejects", "rock4_matvecs",
                                         "rock4_s_min", "rock4_s_max", "rock4_rounds",
                                         "rock4_mat_slots")] + [("rho1", C.c_double), ("rock4_kernel_ms", C.c_double),
                                                          ("reaction_ms", C.c_double), ("diffusion_ms", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def lib():
    """Load librdmr.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_1506_04651_b200.build`")
        L = C.CDLL(LIB_PATH)
        vp, i64, dp = C.c_void_p, C.c_int64, C.c_double
        L.rd_status_string.restype = C.c_char_p
        L.rd_status_string.argtypes = [C.c_int]
        L.mr_grid_build.argtypes = [C.POINTER(mr_params), C.c_int, vp, vp, C.POINTER(vp)]
        L.mr_adapt.argtypes = [vp, vp]
        L.mr_set_operator.argtypes = [vp, C.c_int, vp]
        L.mr_grid_leaves.argtypes = [vp, C.POINTER(i64), C.POINTER(vp), C.POINTER(vp)]
        L.mr_grid_info.argtypes = [vp, C.POINTER(i64), C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(dp),
                                   C.POINTER(dp)]
        L.mr_grid_free.argtypes = [vp]
        L.mr_grid_free.restype = None
        L.mr_key_encode.restype = C.c_uint64
        L.mr_key_encode.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int32)]
        L.mr_key_decode.restype = None
        L.mr_key_decode.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int32)]
        L.mr_rowmajor_to_morton.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, vp]
        L.rd_fv_apply.argtypes = [vp, vp, vp, vp]
        L.rd_reaction_radau5.argtypes = [i64, C.c_int, vp, C.POINTER(rd_model), dp, C.POINTER(rd_radau5_opts),
                                         C.POINTER(rd_stats), vp, vp]
        L.rd_reaction_rk4.argtypes = [i64, C.c_int, vp, C.POINTER(rd_model), dp, C.c_int, vp]
        L.rd_reaction_radau5_cells.argtypes = [i64, i64, C.c_int, vp, C.POINTER(rd_model), dp,
                                               C.POINTER(rd_radau5_opts), vp, C.POINTER(rd_stats), vp, vp]
        L.rd_reaction_cost.argtypes = [i64, i64, C.c_int, vp, C.POINTER(rd_model), C.POINTER(rd_radau5_opts), vp, vp]
        L.rd_shard_bounds.argtypes = [i64, vp, C.c_int, C.POINTER(C.c_int64), vp]
        L.rd_diffusion_rock4.argtypes = [vp, C.POINTER(dp), dp, C.POINTER(rd_rock4_opts), C.POINTER(rd_stats), vp]
        L.rd_rock4_forced_step.argtypes = [vp, vp, dp, dp, C.c_int, vp, vp, vp]
        L.rd_strang_step.argtypes = [vp, C.POINTER(rd_model), C.POINTER(dp), dp, C.c_int,
                                     C.POINTER(rd_radau5_opts), C.POINTER(rd_rock4_opts), C.POINTER(rd_stats), vp]
        L.mr_grid_stats.argtypes = [vp, C.POINTER(i64), C.c_int]
        L.rd_kernel_launches.restype = C.c_int64
        L.rd_kernel_launches.argtypes = []
        L.rd_rock4_smax.restype = C.c_int
        L.rd_rock4_smax.argtypes = []
        L.rd_rock4_coeffs.argtypes = [C.c_int, C.POINTER(dp), C.POINTER(dp), C.POINTER(dp), C.POINTER(dp),
                                      C.POINTER(dp)]
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().rd_status_string(int(s)).decode()


def _check(fn, rc, allow=()):
    if rc != RD_OK and rc not in allow:
        raise RdError(fn, rc)
    return rc


def _ptr(t):
    """Raw device pointer of a contiguous CUDA float64/int tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor required (no CPU path)")
    if not t.is_contiguous():
        raise ValueError("contiguous tensor required")
    return C.c_void_p(t.data_ptr())


def _ptr_rows(t):
    """Raw device pointer of a CUDA 2-D view with unit column stride (row stride = the C ABI's ld)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor required (no CPU path)")
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError("2-D view with unit column stride required")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Model:
    """rd_model with its host arrays kept alive."""

    def __init__(self, spec: dict):
        kind = spec.get("kind", "oregonator")
        self.s = rd_model()
        if kind == "oregonator":
            self.s.kind, self.s.m = RD_MODEL_OREGONATOR, 3
            self.s.q, self.s.f_c = spec.get("q", 2e-3), spec.get("f_c", 1.6)
            self.s.eps_b, self.s.mu = spec.get("eps_b", 1e-2), spec.get("mu", 1e-5)
        elif kind == "nagumo":
            self.s.kind, self.s.m = RD_MODEL_NAGUMO, 1
            self.s.k_nag = spec.get("k", 10.0)
        else:
            self.reac = np.ascontiguousarray(spec["reactants"], dtype=np.int32)
            self.prod = np.ascontiguousarray(spec["products"], dtype=np.int32)
            self.rate = np.ascontiguousarray(spec["rate"], dtype=np.float64)
            self.s.kind = RD_MODEL_MASS_ACTION
            self.s.m = int(spec.get("m", 1 + max(int(self.reac.max()), int(self.prod.max()))))
            self.s.n_reac = len(self.rate)
            self.s.reactants = self.reac.ctypes.data
            self.s.products = self.prod.ctypes.data
            self.s.rate = self.rate.ctypes.data
        self.m = self.s.m


def radau5_opts(rtol=1e-8, atol=1e-8, h0=0.0, nit=7, max_steps=100000):
    o = rd_radau5_opts()
    o.rtol, o.atol, o.h0, o.nit, o.max_steps = rtol, atol, h0, nit, max_steps
    return o


def rock4_opts(rtol=1e-8, atol=1e-8, s_max=200):
    o = rd_rock4_opts()
    o.rtol, o.atol, o.s_max = rtol, atol, s_max
    return o


def rd_reaction_radau5(u, model: Model, T, opts=None, stats=None, cell_counters=None, stream=None,
                       allow_stiff=False):
    """u: CUDA float64 [m, n] (in place).  cell_counters: None or CUDA int32 [8, n]."""
    m, n = u.shape
    rc = lib().rd_reaction_radau5(n, m, _ptr(u), C.byref(model.s), float(T),
                                  C.byref(opts or radau5_opts()), C.byref(stats) if stats is not None else None,
                                  _ptr(cell_counters), _stream(stream))
    return _check("rd_reaction_radau5", rc, (RD_ESTIFF,) if allow_stiff else ())


def rd_reaction_radau5_cells(u, model: Model, T, order=None, opts=None, stats=None, cell_counters=None, stream=None,
                             allow_stiff=False):
    """u: CUDA float64 [m, n] view with unit column stride and row stride ld (e.g. u_full[:, a:b] of a
    [m, N] field: ld = N), in place.  order: None (cells 0..n-1) or CUDA int32 [k] of cell indices in
    [0, n).  cell_counters: None or a CUDA int32 [8, n] view with the same row stride."""
    m, n = u.shape
    ld = max(u.stride(0), n, 1)
    if cell_counters is not None and cell_counters.stride(0) != ld:
        raise ValueError("cell_counters must share u's row stride")
    cnt = n if order is None else order.numel()
    rc = lib().rd_reaction_radau5_cells(cnt, ld, m, _ptr_rows(u), C.byref(model.s), float(T),
                                        C.byref(opts or radau5_opts()), _ptr(order),
                                        C.byref(stats) if stats is not None else None, _ptr_rows(cell_counters),
                                        _stream(stream))
    return _check("rd_reaction_radau5_cells", rc, (RD_ESTIFF,) if allow_stiff else ())


def rd_reaction_cost(u, model: Model, opts=None, stream=None):
    """Cost-proxy keys (CUDA int32 [n]) of the cells of u (CUDA float64 [m, n] view, unit column stride)."""
    import torch
    m, n = u.shape
    ld = max(u.stride(0), n, 1)
    key = torch.empty(n, dtype=torch.int32, device=u.device)
    _check("rd_reaction_cost", lib().rd_reaction_cost(n, ld, m, _ptr_rows(u), C.byref(model.s),
                                                      C.byref(opts or radau5_opts()), _ptr(key), _stream(stream)))
    return key


def rd_shard_bounds(n, cost, p, stream=None):
    """Cost-balanced interval bounds [p + 1] of [0, n) (include/rdmr.h); cost: CUDA int32 [n] or None."""
    b = (C.c_int64 * (p + 1))()
    _check("rd_shard_bounds", lib().rd_shard_bounds(int(n), _ptr(cost), int(p), b, _stream(stream)))
    return list(b)


def rd_reaction_rk4(u, model: Model, T, nsteps=1, stream=None):
    """u: CUDA float64 [m, n] (in place): nsteps equal classical RK4 steps over [0, T] per cell."""
    m, n = u.shape
    rc = lib().rd_reaction_rk4(n, m, _ptr(u), C.byref(model.s), float(T), int(nsteps), _stream(stream))
    return _check("rd_reaction_rk4", rc)


def mr_key_encode(dim, level, k):
    kk = (C.c_int32 * 3)(*(list(k) + [0] * (3 - len(k))))
    return int(lib().mr_key_encode(dim, level, kk))


def mr_key_decode(dim, key):
    lv = C.c_int()
    kk = (C.c_int32 * 3)()
    lib().mr_key_decode(dim, C.c_uint64(key), C.byref(lv), kk)
    return lv.value, tuple(kk[:dim])


def mr_rowmajor_to_morton(dim, level, u_rowmajor, stream=None):
    """u_rowmajor: CUDA float64 [m, 2^{dJ}] (x fastest) -> new tensor in level-J Morton order."""
    import torch
    src = u_rowmajor.reshape(u_rowmajor.shape[0], -1).contiguous()
    dst = torch.empty_like(src)
    _check("mr_rowmajor_to_morton", lib().mr_rowmajor_to_morton(dim, level, src.shape[0], _ptr(src), _ptr(dst),
                                                                _stream(stream)))
    return dst


class Grid:
    """Owning handle of an mr_grid (device resident)."""

    def __init__(self, handle, m, dim):
        self.h, self.m, self.dim = handle, m, dim

    @classmethod
    def build(cls, dim, level_min, level_max, eps_mr, u_finest_morton, stream=None):
        p = mr_params(dim, level_min, level_max, eps_mr)
        h = C.c_void_p()
        m = u_finest_morton.shape[0]
        _check("mr_grid_build", lib().mr_grid_build(C.byref(p), m, _ptr(u_finest_morton), _stream(stream),
                                                    C.byref(h)))
        return cls(h, m, dim)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mr_grid_free(self.h)
            self.h = None

    def adapt(self, stream=None):
        _check("mr_adapt", lib().mr_adapt(self.h, _stream(stream)))

    def set_operator(self, mode, stream=None):
        """RD_OP_PREDICTION (default), RD_OP_TWO_POINT or RD_OP_TWO_POINT_COMPACT (include/rdmr.h)."""
        _check("mr_set_operator", lib().mr_set_operator(self.h, int(mode), _stream(stream)))

    def leaves(self):
        """(n, keys_ptr, u_ptr) raw; see leaf_tensors for torch views."""
        n = C.c_int64()
        kp, up = C.c_void_p(), C.c_void_p()
        _check("mr_grid_leaves", lib().mr_grid_leaves(self.h, C.byref(n), C.byref(kp), C.byref(up)))
        return n.value, kp.value, up.value

    def leaf_tensors(self):
        """Copies of (keys int64 [N], u float64 [m, N]) as CUDA tensors."""
        import torch
        n, kp, up = self.leaves()
        keys = torch.empty(n, dtype=torch.int64, device="cuda")
        u = torch.empty((self.m, n), dtype=torch.float64, device="cuda")
        if n:
            _cuda_memcpy_d2d(keys.data_ptr(), kp, 8 * n)
            _cuda_memcpy_d2d(u.data_ptr(), up, 8 * n * self.m)
        return keys, u

    def values_view(self):
        """Zero-copy CUDA float64 [m, N] view of the grid's leaf values (valid until the next adapt /
        build; writes go straight to the grid)."""
        import torch
        n, _, up = self.leaves()

        class _Iface:
            __cuda_array_interface__ = {"shape": (self.m, n), "typestr": "<f8", "data": (up or 0, False),
                                        "version": 3, "strides": None}
        if n == 0:
            return torch.empty((self.m, 0), dtype=torch.float64, device="cuda")
        return torch.as_tensor(_Iface(), device="cuda")

    def set_values(self, u):
        """Overwrite the leaf state from a CUDA float64 [m, N] tensor."""
        n, _, up = self.leaves()
        assert tuple(u.shape) == (self.m, n)
        u = u.contiguous()
        _cuda_memcpy_d2d(up, u.data_ptr(), 8 * n * self.m)

    def info(self):
        ni, lo, hi, cr, rho = C.c_int64(), C.c_int(), C.c_int(), C.c_double(), C.c_double()
        _check("mr_grid_info", lib().mr_grid_info(self.h, C.byref(ni), C.byref(lo), C.byref(hi), C.byref(cr),
                                                  C.byref(rho)))
        return dict(n_internal=ni.value, level_lo=lo.value, level_hi=hi.value, cr=cr.value, rho1=rho.value)

    def stats(self):
        out = (C.c_int64 * 8)()
        _check("mr_grid_stats", lib().mr_grid_stats(self.h, out, 8))
        return dict(zip(("n_leaves", "n_interface_terms", "n_needed_internal", "n_expansion", "dense_total", "dim",
                         "J", "L_min"), out[:]))

    @property
    def n_leaves(self):
        return self.leaves()[0]

    def fv_apply(self, x, stream=None):
        import torch
        y = torch.empty_like(x)
        _check("rd_fv_apply", lib().rd_fv_apply(self.h, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def diffusion_rock4(self, eps_diff, T, opts=None, stats=None, stream=None):
        eps = (C.c_double * self.m)(*[float(e) for e in eps_diff])
        _check("rd_diffusion_rock4", lib().rd_diffusion_rock4(self.h, eps, float(T), C.byref(opts or rock4_opts()),
                                                              C.byref(stats) if stats is not None else None,
                                                              _stream(stream)))

    def rock4_forced_step(self, x, eps, h, s, stream=None):
        import torch
        out, err = torch.empty_like(x), torch.empty_like(x)
        _check("rd_rock4_forced_step", lib().rd_rock4_forced_step(self.h, _ptr(x), float(eps), float(h), int(s),
                                                                  _ptr(out), _ptr(err), _stream(stream)))
        return out, err

    def strang_step(self, model: Model, eps_diff, dt, scheme=RD_STRANG_RDR, ropts=None, kopts=None, stats=None,
                    stream=None):
        eps = (C.c_double * self.m)(*[float(e) for e in eps_diff])
        rc = lib().rd_strang_step(self.h, C.byref(model.s), eps, float(dt), int(scheme),
                                  C.byref(ropts or radau5_opts()), C.byref(kopts or rock4_opts()),
                                  C.byref(stats) if stats is not None else None, _stream(stream))
        return _check("rd_strang_step", rc)


def _cuda_memcpy_d2d(dst, src, nbytes):
    """Stream-ordered device-to-device copy via the CUDA runtime librdmr.so links (plumbing)."""
    import torch
    L = lib()
    fn = L.cudaMemcpyAsync
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
    rc = fn(C.c_void_p(dst), C.c_void_p(src), C.c_size_t(nbytes), 3, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed ({rc})")


def rock4_coeffs(s):
    n = s - 4
    ell = C.c_double()
    sig = (C.c_double * 4)()
    mu, nu, ka = (C.c_double * n)(), (C.c_double * n)(), (C.c_double * n)()
    _check("rd_rock4_coeffs", lib().rd_rock4_coeffs(s, C.byref(ell), sig, mu, nu, ka))
    return dict(s=s, ell=ell.value, sigma=np.array(sig[:]), mu=np.array(mu[:]), nu=np.array(nu[:]),
                kappa=np.array(ka[:]))


def kernel_launches():
    return int(lib().rd_kernel_launches())


def rock4_smax():
    return int(lib().rd_rock4_smax())
