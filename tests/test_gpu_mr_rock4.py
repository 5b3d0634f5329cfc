"""GPU parity of the MR grid (build / adapt: bit-exact leaf sets, keys and values; P:537-625,
841-938), the FV operator (rd_fv_apply), Rock4 (forced step + controlled integration,
P:957-997) and the Strang step against the oracle, through the C-ABI."""
import numpy as np
import pytest

import synth
from tests.grids import front_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def gpu_build(P, dim, lmin, J, eps, u_rowmajor):
    import torch
    ut = torch.tensor(np.ascontiguousarray(u_rowmajor.reshape(u_rowmajor.shape[0], -1)), device="cuda")
    um = P.mr_rowmajor_to_morton(dim, J, ut)
    return P.Grid.build(dim, lmin, J, eps, um)


def gpu_leaves(g):
    keys, u = g.leaf_tensors()
    return keys.cpu().numpy().view(np.uint64), u.cpu().numpy()


def assert_same_grid(g, o):
    gk, gu = gpu_leaves(g)
    ok, ou = o.leaves()
    assert len(gk) == len(ok), (len(gk), len(ok))
    assert np.array_equal(gk, ok)
    assert np.array_equal(gu, ou)  # projections / predictions are bit-exact (FMA-free, same order)


CASES = [(2, 2, 6, 1e-2, 1), (2, 3, 7, 3e-3, 3), (2, 0, 5, 5e-2, 2), (3, 1, 4, 1e-2, 1), (3, 2, 5, 2e-2, 3)]


@pytest.mark.parametrize("dim,lmin,J,eps,m", CASES)
def test_build_bit_exact(P, orc, dim, lmin, J, eps, m):
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    assert_same_grid(g, o)
    info = g.info()
    assert info["rho1"] == o.rho1
    n = g.n_leaves
    assert info["cr"] == pytest.approx(1 - n / 2 ** (dim * J))


@pytest.mark.parametrize("dim,lmin,J", [(2, 3, 6), (3, 2, 4)])
def test_eps_zero_is_uniform(P, orc, dim, lmin, J):
    """eps = 0 => uniform level J, bit-for-bit the Morton-ordered input (BJ north_star)."""
    u = front_field(dim, J, 2)
    g = gpu_build(P, dim, lmin, J, 0.0, u)
    k, v = gpu_leaves(g)
    assert len(k) == 2 ** (dim * J)
    assert all(int(x) >> 58 == J for x in k[:: max(1, len(k) // 97)])
    o = orc.Grid.build(dim, lmin, J, 0.0, u.reshape(2, -1))
    assert_same_grid(g, o)


@pytest.mark.parametrize("dim,lmin,J,eps,m", CASES)
def test_adapt_bit_exact(P, orc, dim, lmin, J, eps, m):
    """Build, move the field, adapt three times: identical leaf sets and values after every call."""
    import torch
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    for it in range(3):
        keys, vals = o.leaves()
        lv = np.array([int(x) >> 58 for x in keys])
        # new leaf values: a moved front evaluated at leaf centres (same values on both sides)
        from tests.mr_ref import morton_decode
        cen = np.array([[(c + 0.5) * 2.0 ** -j for c in morton_decode(dim, int(kk))[1]] for kk, j in zip(keys, lv)])
        shift = 0.06 * (it + 1)
        r = np.sqrt(((cen - np.array([0.4 + shift, 0.55, 0.5][:dim])) ** 2).sum(1))
        newv = vals.copy()
        newv[0] = np.tanh((0.25 - r) / 0.03)
        o.set_values(newv)
        g.set_values(torch.tensor(newv, device="cuda"))
        o.adapt()
        g.adapt()
        assert_same_grid(g, o)
        assert o.check() == 0
        assert g.info()["rho1"] == o.rho1


def test_cfg3_build_calibration(P, orc):
    """BJ configs[2] build: "roughly 1e5 to 2e5 leaves" (BJ); 152 806 with radius-2 grading (DESIGN.md
    R-G2; SURVEY's 144 388 probe used radius 1), identical to the oracle."""
    w = synth.cfg3()
    g = gpu_build(P, 2, w.level_min, w.level_max, w.eps_mr, w.u)
    assert g.n_leaves == 152806
    o = orc.Grid.build(2, w.level_min, w.level_max, w.eps_mr, w.u.reshape(3, -1))
    assert_same_grid(g, o)


def test_cfg4_build_calibration(P, orc):
    """BJ configs[3] build: "~1e6 leaves" (BJ), identical to the oracle (radius-2 grading, R-G2)."""
    w = synth.cfg4()
    g = gpu_build(P, 3, w.level_min, w.level_max, w.eps_mr, w.u)
    assert g.n_leaves == 1071519  # oracle count (BJ "~1e6 leaves")
    o = orc.Grid.build(3, w.level_min, w.level_max, w.eps_mr, w.u.reshape(3, -1))
    assert_same_grid(g, o)


@pytest.mark.parametrize("dim,lmin,J,eps,m", CASES[:4])
def test_fv_apply(P, orc, dim, lmin, J, eps, m, r4mode):
    """A x on the leaves vs the oracle's operator (O.5), in both operator forms: the assembled leaf
    matrix (prediction + projection weights folded in, FP32-exact weights) and the matrix-free stencil."""
    import torch
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    rng = np.random.default_rng(3)
    x = rng.standard_normal(g.n_leaves)
    y = g.fv_apply(torch.tensor(x, device="cuda")).cpu().numpy()
    yo = o.apply(x)
    scale = np.abs(yo).max()
    assert np.max(np.abs(y - yo)) <= 1e-12 * scale
    # conservation: sum |C| (Ax)_C = 0 (Neumann)
    keys, _ = gpu_leaves(g)
    vol = np.array([2.0 ** (-dim * (int(k) >> 58)) for k in keys])
    assert abs((vol * y).sum()) <= 1e-12 * (vol * np.abs(y)).sum()


@pytest.fixture(params=["mat", "free"])
def r4mode(request, monkeypatch):
    """Rock4 operator form: the assembled sparse leaf operator (2-D default, fvmat.cu) or the
    matrix-free stencil with per-stage projection / ghost phases (3-D default)."""
    monkeypatch.setenv("RDMR_R4_MODE", request.param)
    return request.param


@pytest.mark.parametrize("s", [5, 7, 12, 25])
def test_rock4_forced_eigenmode(P, s, r4mode):
    """Forced step on a Neumann eigenmode of the 128^2 uniform grid: out = R_s(h lam) v (BJ north_star)."""
    import torch
    J, dim = 7, 2
    n = 1 << J
    k1, k2 = 3, 5
    xx = (np.arange(n) + 0.5) / n
    v = np.outer(np.cos(np.pi * k2 * xx), np.cos(np.pi * k1 * xx))  # rows y, cols x
    g = gpu_build(P, dim, J, J, 0.0, v[None])
    eps = 2.5e-3
    lam = -eps * 4 * n * n * (np.sin(np.pi * k1 / (2 * n)) ** 2 + np.sin(np.pi * k2 / (2 * n)) ** 2)
    c = P.rock4_coeffs(s)
    h = 0.9 * c["ell"] / (eps * g.info()["rho1"])
    _, vm = gpu_leaves(g)
    out, err = g.rock4_forced_step(torch.tensor(vm[0], device="cuda"), eps, h, s)
    z = h * lam
    # R_s(z) = w(z) P_n(z) from the library's own coefficients
    Pm, Pc = 0.0, 1.0
    for mu, nu, ka in zip(c["mu"], c["nu"], c["kappa"]):
        Pm, Pc = Pc, (nu + mu * z) * Pc + ka * Pm
    sg = c["sigma"]
    R = (1 + z * (sg[0] + z * (sg[1] + z * (sg[2] + z * sg[3])))) * Pc
    # DESIGN.md reading R-K6: rounding of the s recurrence stages leaves O(s eps_mach |v|) noise on
    # every mode of g_{s-4}; the finishing polynomial w multiplies it by up to max |w| on [-ell, 0]
    # (1.7e1 at s = 5, 2.2e7 at s = 25), so |out - R v| <= C s eps_mach max|w| |v|.  Observed C <= 0.05
    # on both operator forms (tools/r4_forced_err.py, s = 5..40); the test allows C = 0.25.
    zz = -np.linspace(0, c["ell"], 4001)
    wmax = np.abs(1 + zz * (sg[0] + zz * (sg[1] + zz * (sg[2] + zz * sg[3])))).max()
    tol = 4e-16 + 0.25 * np.finfo(float).eps * s * wmax
    assert np.max(np.abs(out.cpu().numpy() - R * vm[0])) <= tol
    assert np.max(np.abs(err.cpu().numpy() - sg[3] * z ** 4 * Pc * vm[0])) <= tol


def test_rock4_table_vs_oracle_table(P, orc):
    """The coefficients the kernel uses (rd_rock4_coeffs) against the oracle's generator evaluated at
    the same ell (independent fixed-point implementations, R-K1); ell itself within 1e-4."""
    from oracle import rock4_family as F
    assert P.rock4_smax() == 200
    for s in range(5, P.rock4_smax() + 1, 13):
        a, b = P.rock4_coeffs(s), orc.rock4_coeffs(s)
        assert a["ell"] == pytest.approx(b["ell"], rel=1e-4)
        ok, sig, mu, nu, ka = F.fixed_point(s, a["ell"])
        assert ok
        assert np.allclose(a["sigma"], sig, rtol=1e-9, atol=1e-14)
        assert np.allclose(a["mu"], mu, rtol=1e-9, atol=1e-16)


@pytest.mark.parametrize("dim,lmin,J,eps,T", [(2, 7, 7, 0.0, 1e-3), (2, 3, 7, 3e-3, 1e-3), (2, 2, 6, 1e-2, 1e-2),
                                             (3, 2, 5, 2e-2, 1e-3)])
def test_diffusion_rock4_vs_oracle(P, orc, dim, lmin, J, eps, T, r4mode):
    """Controlled Rock4 on the leaves vs the oracle: normwise relative error <= 1e-6 per species."""
    m = 3
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    epsd = [2.5e-3, 2.5e-3, 1.5e-3]
    st = P.rd_stats()
    g.diffusion_rock4(epsd, T, stats=st)
    ost = o.diffuse(epsd, T)
    _, gu = gpu_leaves(g)
    _, ou = o.leaves()
    err = np.abs(gu - ou).max(1) / np.abs(ou).max(1)
    assert (err <= 1e-6).all(), err
    assert st.rock4_steps >= 3 and st.rock4_matvecs > 0
    # the requested operator form ran (3-D rows may exceed the assembled row cap: then matrix-free)
    if r4mode == "free":
        assert st.rock4_mat_slots == 0
    elif dim == 2:
        assert st.rock4_mat_slots >= len(gu[0])
    # mass conservation (Neumann)
    keys, _ = gpu_leaves(g)
    vol = np.array([2.0 ** (-dim * (int(k) >> 58)) for k in keys])
    u0 = P  # noqa
    assert np.allclose((gu * vol).sum(1), (ou * vol).sum(1), rtol=1e-12)


@pytest.mark.parametrize("dim,lmin,J,eps", [(2, 3, 7, 3e-3), (3, 2, 5, 2e-2)])
def test_diffusion_rock4_consecutive_calls(P, orc, dim, lmin, J, eps, r4mode):
    """Three consecutive D substeps on the same grids (reading R-K5b: each species' controller starts from
    the step size it proposed when the previous substep ended, h0 = T on a fresh grid): the states stay
    within 1e-6 of the oracle after every call, both sides take the same accepted-step counts, and the
    warm-started calls reject fewer steps than the cold first call."""
    m = 3
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    epsd = [2.5e-3, 2.5e-3, 1.5e-3]
    T = 1e-2  # long enough that the cold h0 = T is rejected (oracle: 2-D 2 rejects, 3-D 1, then none)
    rej = []
    for call in range(3):
        st = P.rd_stats()
        g.diffusion_rock4(epsd, T, stats=st)
        ost = o.diffuse(epsd, T)
        _, gu = gpu_leaves(g)
        _, ou = o.leaves()
        err = np.abs(gu - ou).max(1) / np.abs(ou).max(1)
        assert (err <= 1e-6).all(), (call, err)
        assert st.rock4_steps == ost["steps"] and st.rock4_rejects == ost["rejects"], (call, st.rock4_steps, ost)
        rej.append(st.rock4_rejects)
    assert rej[0] >= 1 and rej[1] < rej[0] and rej[2] < rej[0], rej


@pytest.mark.parametrize("m", [2, 4, 5])
def test_diffusion_rock4_species_counts(P, orc, m, r4mode):
    """Species counts that leave a remainder after the kernels' groups of 3 (2, 4 -> 3 + 1, 5 -> 3 + 2),
    with per-species eps so that the species' step sequences (and rejections) desynchronise."""
    dim, lmin, J, eps, T = 2, 3, 7, 3e-3, 3e-3
    u = front_field(dim, J, m)
    g = gpu_build(P, dim, lmin, J, eps, u)
    o = orc.Grid.build(dim, lmin, J, eps, u.reshape(m, -1))
    epsd = [2.5e-3 * (1 + 0.7 * i) for i in range(m)]
    g.diffusion_rock4(epsd, T)
    o.diffuse(epsd, T)
    _, gu = gpu_leaves(g)
    _, ou = o.leaves()
    err = np.abs(gu - ou).max(1) / np.abs(ou).max(1)
    assert (err <= 1e-6).all(), err


def _strang_parity(P, orc, w, steps, scheme=0, adapt=True, resync=False):
    """`steps` Strang steps on the GPU and in the oracle from the same initial data; after every step the
    leaf sets must be identical and the states within 1e-6 normwise per species (S20).  With adapt (or
    resync) both continue from the SAME state (the GPU's), so parity is checked per step."""
    import os
    import torch
    dim, J = w.dim, w.level_max
    g = gpu_build(P, dim, w.level_min, J, w.eps_mr, w.u)
    o = orc.Grid.build(dim, w.level_min, J, w.eps_mr, w.u.reshape(w.m, -1))
    spec = dict(w.model, m=w.m)
    gm, om = P.Model(spec), orc.Model(spec)
    worst = 0.0
    for it in range(steps):
        g.strang_step(gm, w.eps_diff, w.dt, scheme)
        rc = o.strang(om, w.eps_diff, w.dt, scheme, nthreads=os.cpu_count() or 16)
        assert rc == 0
        gk, gu = gpu_leaves(g)
        ok, ou = o.leaves()
        assert np.array_equal(gk, ok)
        err = np.abs(gu - ou).max(1) / np.abs(ou).max(1)
        worst = max(worst, err.max())
        assert (err <= 1e-6).all(), (it, err)
        if adapt or resync:
            # continue both from the SAME state (the GPU's) so leaf-set parity is per call
            o.set_values(gu)
            g.set_values(torch.tensor(gu, device="cuda"))
        if adapt:
            o.adapt()
            g.adapt()
            assert_same_grid(g, o)
    return worst


def test_strang_cfg1(P, orc):
    """BJ configs[0]: uniform 128^2 BZ, one RDR step dt = 1e-3 (full size)."""
    _strang_parity(P, orc, synth.cfg1(), 1, adapt=False)


def test_strang_cfg1_drd(P, orc):
    _strang_parity(P, orc, synth.cfg1(), 1, scheme=1, adapt=False)


def test_strang_cfg3_five_steps(P, orc):
    """BJ configs[2] (full size: J=10, 1.5e5 leaves): 5 Strang steps, each followed by re-adaptation."""
    _strang_parity(P, orc, synth.cfg3(), 5)


@pytest.mark.slow
def test_strang_cfg4_two_steps(P, orc):
    """BJ configs[3] (full size 3-D, ~1.07e6 leaves): 2 Strang steps, each followed by re-adaptation."""
    _strang_parity(P, orc, synth.cfg4(), 2)


@pytest.mark.slow
def test_strang_cfg5_full_step(P, orc):
    """BJ configs[4] at full size: 512^2 uniform, the m = 20 mass-action network (warp-per-cell Radau5
    on all 262 144 cells) and 20-species Rock4 in one persistent kernel: one RDR Strang step, dt = 1e-4,
    against the threaded oracle (~3 min of host time)."""
    _strang_parity(P, orc, synth.cfg5(), 1, adapt=False)


def test_strang_small_3d(P, orc):
    w = synth.cfg4(J=5, K=3)
    _strang_parity(P, orc, w, 2)


def test_strang_drd_mr(P, orc):
    """DRD variant on an adaptive 2-D grid, with re-adaptation."""
    w = synth.cfg3(J=8, K=3)
    _strang_parity(P, orc, w, 2, scheme=1)


def test_strang_cfg5_reduced(P, orc):
    """BJ configs[4]'s m = 20 network and diffusion on a 64^2 grid (J = 6): warp-per-cell Radau5 + Rock4
    with 20 species in one persistent kernel, 2 Strang steps vs the oracle."""
    w = synth.cfg5(J=6)
    _strang_parity(P, orc, w, 2, adapt=False)


def test_adapt_degenerate_cases(P, orc):
    """L_min = J (nothing may coarsen), a huge threshold (everything coarsens to L_min), and a
    constant field (all details zero): identical to the oracle and graded."""
    import torch
    for (dim, lmin, J, eps) in [(2, 5, 5, 1e-2), (2, 2, 6, 1e3), (3, 1, 4, 1e3)]:
        u = front_field(dim, J, 2)
        g = gpu_build(P, dim, lmin, J, eps, u)
        o = orc.Grid.build(dim, lmin, J, eps, u.reshape(2, -1))
        assert_same_grid(g, o)
        if eps >= 1e3:
            assert g.n_leaves == 2 ** (dim * lmin)
        g.adapt()
        o.adapt()
        assert_same_grid(g, o)
    c = np.ones((1, 1 << 10)) * 0.7
    g = gpu_build(P, 2, 1, 5, 1e-6, c)
    assert g.n_leaves == 4  # constant field: zero details, coarsens to L_min = 1
    k, v = gpu_leaves(g)
    assert np.all(v == 0.7)


def test_grid_api_errors(P):
    """Invalid arguments return RD_EINVAL and create nothing (include/rdmr.h conventions)."""
    import ctypes as C
    import torch
    L = P.lib()
    u = torch.zeros(4 ** 5, dtype=torch.float64, device="cuda")
    h = C.c_void_p()
    for prm in [P.mr_params(4, 1, 5, 0.0), P.mr_params(2, 6, 5, 0.0), P.mr_params(2, 1, 15, 0.0),
                P.mr_params(3, 1, 10, 0.0), P.mr_params(2, 1, 5, -1.0)]:
        assert L.mr_grid_build(C.byref(prm), 1, C.c_void_p(u.data_ptr()), None, C.byref(h)) == P.RD_EINVAL
    prm = P.mr_params(2, 1, 5, 0.0)
    assert L.mr_grid_build(C.byref(prm), 0, C.c_void_p(u.data_ptr()), None, C.byref(h)) == P.RD_EINVAL
    assert L.mr_grid_build(C.byref(prm), 1, None, None, C.byref(h)) == P.RD_EINVAL
    assert L.mr_adapt(None, None) == P.RD_EINVAL
    g = P.Grid.build(2, 1, 5, 0.0, u.view(1, -1))
    x = torch.zeros(g.n_leaves, dtype=torch.float64, device="cuda")
    assert L.rd_fv_apply(g.h, C.c_void_p(x.data_ptr()), C.c_void_p(x.data_ptr()), None) == P.RD_EINVAL
    assert L.rd_rock4_forced_step(g.h, C.c_void_p(x.data_ptr()), 1.0, 1e-3, 4, C.c_void_p(x.data_ptr()), None,
                                  None) == P.RD_EINVAL
    eps = (C.c_double * 1)(-1.0)
    assert L.rd_diffusion_rock4(g.h, eps, 1e-3, None, None, None) == P.RD_EINVAL


def test_diffusion_zero_eps_is_identity(P):
    """D with eps = 0 leaves the species unchanged (Strang degeneracy eps = 0, SURVEY pins)."""
    import torch
    u = front_field(2, 6, 3)
    g = gpu_build(P, 2, 2, 6, 1e-2, u)
    _, before = gpu_leaves(g)
    g.diffusion_rock4([0.0, 2.5e-3, 0.0], 1e-3)
    _, after = gpu_leaves(g)
    assert np.array_equal(before[0], after[0]) and np.array_equal(before[2], after[2])
    assert not np.array_equal(before[1], after[1])


@pytest.mark.parametrize("strict", [True, False])
def test_coarsen_threshold_tie_gpu(P, orc, strict):
    """P:590-596 / reading S12 on the GPU: Q = E_J exactly keeps the finest cells (coarsen only when
    SMALLER), one part in 2^20 less coarsens them; same leaf set as the oracle."""
    from tests.test_oracle_mr import _tie_field
    J, eps = 5, 2.0 ** -4
    amp = 2.0 ** -4 if strict else 2.0 ** -4 * (1 - 2.0 ** -20)
    u = _tie_field(J, amp, J)
    g = gpu_build(P, 2, 1, J, eps, u)
    o = orc.Grid.build(2, 1, J, eps, u.reshape(1, -1))
    assert_same_grid(g, o)
    gk, _ = gpu_leaves(g)
    assert ((gk >> np.uint64(58)) == J).any() == strict


@pytest.mark.parametrize("tie", [True, False])
def test_refine_threshold_tie_gpu(P, orc, tie):
    """P:590-596 / reading S12 on the GPU: a leaf with Q = E_j exactly is not refined (refine only when
    the detail EXCEEDS the threshold); one part in 2^20 more refines it; same leaf set as the oracle."""
    from tests.test_oracle_mr import _tie_field
    J, eps = 5, 2.0 ** -4
    amp = 2.0 ** -5 if tie else 2.0 ** -5 * (1 + 2.0 ** -20)
    u = _tie_field(J, amp, J - 1)
    g = gpu_build(P, 2, J - 1, J, eps, u)
    o = orc.Grid.build(2, J - 1, J, eps, u.reshape(1, -1))
    g.adapt()
    o.adapt()
    assert_same_grid(g, o)
    gk, _ = gpu_leaves(g)
    assert ((gk >> np.uint64(58)) == J).any() == (not tie)


def test_rock4_nonfinite_state_fails_fast(P):
    """A non-finite stage value makes the error norm NaN: the species fails at once with RD_ESTIFF
    (include/rdmr.h: failure is reported, no silent clipping) instead of retrying ever larger steps."""
    import time
    import torch
    u = front_field(2, 6, 1)
    g = gpu_build(P, 2, 6, 6, 0.0, u)
    _, v = g.leaf_tensors()
    v[0, 100] = float("nan")
    g.set_values(v)
    t0 = time.time()
    with pytest.raises(P.RdError) as ei:
        g.diffusion_rock4([2.5e-3], 1e-3)
    torch.cuda.synchronize()
    assert ei.value.status == P.RD_ESTIFF
    assert time.time() - t0 < 10.0
