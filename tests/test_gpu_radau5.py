"""GPU parity of rd_reaction_radau5 (thread-per-cell and warp-per-cell kernels) against the
oracle's Radau5 (reading O.3), through the C-ABI.  Bar (BJ north_star, DESIGN.md R-P): normwise
max_k |g - o| / max_k |o| <= 1e-6 per species; the step sequences themselves are not compared
(many controllers meet the tolerance)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

TOL = 1e-6


def _normwise(g, o):
    return np.max(np.abs(g - o), axis=1) / np.maximum(np.max(np.abs(o), axis=1), 1e-300)


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def _gpu(P, u, spec, T, **kw):
    import torch
    model = P.Model(spec)
    ut = torch.tensor(u, dtype=torch.float64, device="cuda").contiguous()
    cnt = torch.zeros((8, u.shape[1]), dtype=torch.int32, device="cuda")
    st = P.rd_stats()
    rc = P.rd_reaction_radau5(ut, model, T, P.radau5_opts(**kw), stats=st, cell_counters=cnt,
                              allow_stiff=kw.get("max_steps", 100000) < 100)
    torch.cuda.synchronize()
    return ut.cpu().numpy(), cnt.cpu().numpy(), st, rc


@pytest.mark.parametrize("n", [1, 31, 1000, 4099])
def test_cfg2_cells_small(P, orc, n):
    """cfg-2 recipe cells (several warps + ragged tail) vs the oracle, all cells compared."""
    u0 = synth.random_bz_cells(n, seed=11)
    spec = dict(kind="oregonator", **synth.OREGONATOR)
    g, cnt, st, _ = _gpu(P, u0, spec, 1e-2)
    o, ocnt, ost = orc.radau5(u0, orc.Model(spec), 1e-2, nthreads=8)
    assert (ost == 0).all() and st.n_failed == 0
    assert st.n_cells == n
    err = _normwise(g, o)
    assert (err <= TOL).all(), err
    # counters are per-cell and consistent: f evals >= 1 + 3 * newton, every cell took >= 1 step
    assert (cnt[1] >= 1).all() and (cnt[3] >= 1 + 3 * cnt[6]).all()
    assert st.n_f == int(cnt[3].sum()) and st.n_accept == int(cnt[1].sum())


def test_cfg2_full_size_sampled(P, orc):
    """Full BJ configs[1] (2^22 cells, the bench launch) and 3000 sampled cells recomputed by the oracle."""
    import torch
    w = synth.cfg2()
    spec = w.model
    model = P.Model(spec)
    ut = torch.tensor(w.u, device="cuda")
    st = P.rd_stats()
    P.rd_reaction_radau5(ut, model, 1e-2, stats=st)
    g = ut.cpu().numpy()
    assert st.n_cells == w.u.shape[1] and st.n_failed == 0
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(w.u.shape[1], 3000, replace=False))
    o, _, ost = orc.radau5(w.u[:, idx], orc.Model(spec), 1e-2, nthreads=8)
    assert (ost == 0).all()
    err = _normwise(g[:, idx], o)
    assert (err <= TOL).all(), err
    assert np.isfinite(g).all()


def test_paper_q002(P, orc):
    """The paper's own q = 0.02."""
    u0 = synth.random_bz_cells(500, seed=12)
    spec = dict(kind="oregonator", q=0.02, f_c=1.6, eps_b=1e-2, mu=1e-5)
    g, _, _, _ = _gpu(P, u0, spec, 5e-4)
    o, _, _ = orc.radau5(u0, orc.Model(spec), 5e-4, nthreads=8)
    assert (_normwise(g, o) <= TOL).all()


def test_minimum_complexity(P):
    """A cell at the BZ steady state over T = 5e-4: 1 step, 1 Newton iteration, n_f = 5."""
    q, fc = 2e-3, 1.6
    b = (-(fc + q - 1) + np.sqrt((fc + q - 1) ** 2 + 4 * q * (fc + 1))) / 2
    a = fc * b / (q + b)
    u0 = np.array([[a], [b], [b]])
    g, cnt, _, _ = _gpu(P, u0, dict(kind="oregonator", q=q, f_c=fc, eps_b=1e-2, mu=1e-5), 5e-4)
    att, acc, rej, nf, njac, nlu, nnewt, stat = cnt[:, 0]
    assert (acc, rej, nnewt, nf, njac, nlu) == (1, 0, 1, 5, 1, 1)
    assert np.allclose(g[:, 0], u0[:, 0], rtol=1e-9)


@pytest.mark.parametrize("m,n_reac,seed,n", [(3, 6, 21, 300), (4, 8, 22, 300), (20, 40, 5, 96), (7, 12, 23, 64),
                                             (13, 30, 24, 64), (32, 60, 25, 40)])
def test_mass_action(P, orc, m, n_reac, seed, n):
    """Mass-action networks (BJ configs[4] generator): m <= 4 thread kernel, m > 4 warp kernel (incl.
    padded M and m = 32 lanes), vs the oracle on random positive states."""
    rng = synth.SplitMix64(seed)
    reac, prod, rate = synth.mass_action_network(rng, m, n_reac)
    spec = dict(kind="mass_action", m=m, reactants=reac, products=prod, rate=rate)
    u0 = synth.random_positive_cells(n, m, seed + 100)
    T = 5e-5 if m == 20 else 1e-4
    g, cnt, st, _ = _gpu(P, u0, spec, T)
    o, _, ost = orc.radau5(u0, orc.Model(spec), T, nthreads=8)
    assert (ost == 0).all() and st.n_failed == 0
    err = _normwise(g, o)
    assert (err <= TOL).all(), err


def test_cfg5_network_cells(P, orc):
    """The cfg-5 network itself on cells of its initial field, over one Strang half step."""
    w = synth.cfg5()
    u0 = w.u.reshape(20, -1)[:, ::997][:, :200].copy()
    g, _, st, _ = _gpu(P, u0, w.model, 0.5 * w.dt)
    o, _, ost = orc.radau5(u0, orc.Model(dict(w.model, m=20)), 0.5 * w.dt, nthreads=8)
    assert (ost == 0).all() and st.n_failed == 0
    assert (_normwise(g, o) <= TOL).all()


def test_edge_cases(P):
    import torch
    model = P.Model(dict(kind="oregonator", **synth.OREGONATOR))
    empty = torch.zeros((3, 0), dtype=torch.float64, device="cuda")
    assert P.rd_reaction_radau5(empty, model, 1e-3) == P.RD_OK
    u = torch.tensor(synth.random_bz_cells(64, 3), device="cuda")
    import ctypes as C
    L = P.lib()
    # invalid arguments: nothing enqueued, RD_EINVAL
    assert L.rd_reaction_radau5(64, 3, C.c_void_p(u.data_ptr()), C.byref(model.s), -1.0, None, None, None,
                                None) == P.RD_EINVAL
    assert L.rd_reaction_radau5(64, 4, C.c_void_p(u.data_ptr()), C.byref(model.s), 1e-3, None, None, None,
                                None) == P.RD_EINVAL
    bad = P.radau5_opts(rtol=0.0)
    assert L.rd_reaction_radau5(64, 3, C.c_void_p(u.data_ptr()), C.byref(model.s), 1e-3, C.byref(bad), None, None,
                                None) == P.RD_EINVAL


def test_stiff_failure_reported(P):
    """max_steps too small: RD_ESTIFF, n_failed counted, failed cells keep a finite accepted state."""
    u0 = synth.random_bz_cells(256, seed=13)
    g, cnt, st, rc = _gpu(P, u0, dict(kind="oregonator", **synth.OREGONATOR), 1e-2, max_steps=3)
    assert rc == P.RD_ESTIFF
    assert st.n_failed > 0
    assert np.isfinite(g).all()


def test_complexity_counters_vs_oracle(P, orc):
    """Per-node complexity (n_f + 3 n_jac) from the GPU counters against the
    oracle's on cfg-3 fronts over dt/2: the Newton / step heuristics run in FP32 on the GPU,
    so a few nodes may take another step sequence; the distributions must agree."""
    import torch
    w = synth.cfg3(J=8)
    u0 = w.u.reshape(3, -1)[:, ::7].copy()
    n = u0.shape[1]
    cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")
    P.rd_reaction_radau5(torch.tensor(u0, device="cuda"), P.Model(w.model), 0.5 * w.dt, cell_counters=cnt)
    g = cnt.cpu().numpy().astype(np.int64)
    _, oc, st = orc.radau5(u0, orc.Model(w.model), 0.5 * w.dt, nthreads=8)
    assert (st == 0).all()
    cg, co = g[3] + 3 * g[4], oc[3] + 3 * oc[4]
    assert (cg == co).mean() >= 0.95
    assert abs(cg.mean() - co.mean()) <= 0.02 * co.mean()
    assert cg.min() == co.min() and np.median(cg) == np.median(co)


def test_concurrent_calls_on_two_streams(P):
    """Two rd_reaction_radau5 calls running at the same time on two streams (two host threads; ctypes
    releases the GIL) each have their own work counter and totals (per-call scratch): both results equal
    the sequential ones bit for bit, and each call's stats count exactly its own cells."""
    import threading
    import torch
    spec = dict(kind="oregonator", **synth.OREGONATOR)
    M = P.Model(spec)
    ua = torch.tensor(synth.random_bz_cells(300000, seed=21), device="cuda")
    ub = torch.tensor(synth.random_bz_cells(200000, seed=22), device="cuda")
    ra, rb = ua.clone(), ub.clone()
    P.rd_reaction_radau5(ra, M, 1e-2)
    P.rd_reaction_radau5(rb, M, 1e-2)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    sta, stb = P.rd_stats(), P.rd_stats()
    errs = []

    def run(u, st, stream):
        try:
            P.rd_reaction_radau5(u, M, 1e-2, stats=st, stream=stream)
        except Exception as e:  # noqa: BLE001 (reported below)
            errs.append(e)

    ta = threading.Thread(target=run, args=(ua, sta, sa))
    tb = threading.Thread(target=run, args=(ub, stb, sb))
    ta.start(); tb.start(); ta.join(); tb.join()
    torch.cuda.synchronize()
    assert not errs, errs
    assert torch.equal(ua, ra) and torch.equal(ub, rb)
    assert sta.n_cells == 300000 and stb.n_cells == 200000


def test_mass_action_closed_forms_gpu(P, orc):
    """The thread kernel's mass-action instantiations (m = 2, 3) against closed forms: 2A -> B,
    a(t) = a0 / (1 + 2 k a0 t); A -> B -> C (Bateman).  Tolerances 1e-11 -> relative error <= 1e-8."""
    import torch
    k = 40.0
    spec = dict(kind="mass_action", m=2, reactants=np.array([[0, 0]]), products=np.array([[1, -1]]),
                rate=np.array([k]))
    a0 = np.linspace(0.1, 2.0, 1000)
    u0 = np.stack([a0, np.full_like(a0, 0.25)])
    g, _, st, _ = _gpu(P, u0, spec, 0.3, rtol=1e-11, atol=1e-11)
    a = a0 / (1 + 2 * k * a0 * 0.3)
    assert np.allclose(g[0], a, rtol=1e-8, atol=0) and np.allclose(g[1], 0.25 + (a0 - a) / 2, rtol=1e-8, atol=0)
    k1, k2 = 3.0, 1.2
    spec = dict(kind="mass_action", m=3, reactants=np.array([[0, -1], [1, -1]]), products=np.array([[1, -1], [2, -1]]),
                rate=np.array([k1, k2]))
    u0 = np.tile(np.array([[1.0], [0.0], [0.0]]), (1, 257))
    g, _, st, _ = _gpu(P, u0, spec, 1.0, rtol=1e-11, atol=1e-11)
    A = np.exp(-k1)
    B = k1 / (k2 - k1) * (np.exp(-k1) - np.exp(-k2))
    assert np.allclose(g, np.array([[A], [B], [1 - A - B]]), rtol=1e-8, atol=1e-12)


def test_longest_first_order_leaves_every_cell_unchanged(P, monkeypatch):
    """The plain call schedules >= 65536 cells longest-first by the cost proxy (radau5.cu); the order only
    decides which lane takes which cell, so states and per-cell counters are bit-identical with the
    natural order (RDMR_NO_PROXY_LPT=1) and with an explicit reversed cell list."""
    import torch
    n = 70001  # above the 65536-cell gate, ragged
    u0 = torch.tensor(synth.random_bz_cells(n, seed=5), dtype=torch.float64, device="cuda").contiguous()
    model = P.Model(dict(kind="oregonator", **synth.OREGONATOR))

    def run(order=None):
        u = u0.clone()
        cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")
        st = P.rd_stats()
        if order is None:
            P.rd_reaction_radau5(u, model, 1e-3, stats=st, cell_counters=cnt)
        else:
            P.rd_reaction_radau5_cells(u, model, 1e-3, order=order, stats=st, cell_counters=cnt)
        torch.cuda.synchronize()
        return u, cnt, st

    monkeypatch.delenv("RDMR_NO_PROXY_LPT", raising=False)
    u_lpt, c_lpt, s_lpt = run()
    monkeypatch.setenv("RDMR_NO_PROXY_LPT", "1")
    u_nat, c_nat, s_nat = run()
    u_rev, c_rev, _ = run(torch.arange(n - 1, -1, -1, dtype=torch.int32, device="cuda"))
    assert s_lpt.n_cells == n and s_nat.n_cells == n and s_lpt.n_failed == 0
    assert torch.equal(u_lpt, u_nat) and torch.equal(c_lpt, c_nat)
    assert torch.equal(u_rev, u_nat) and torch.equal(c_rev, c_nat)
    assert s_lpt.n_attempts == s_nat.n_attempts and s_lpt.n_newton == s_nat.n_newton
    assert not torch.equal(u_lpt, u0)


def test_longest_first_order_on_a_strided_interval(P):
    """An interval [a, b) of a wider field (row stride ld > n) with >= 65536 cells goes through the same
    internal longest-first order: bit-identical to the whole-field call on those cells, and the cells
    outside the interval are untouched."""
    import torch
    N, a, b = 140000, 30000, 110001
    u0 = torch.tensor(synth.random_bz_cells(N, seed=9), dtype=torch.float64, device="cuda").contiguous()
    model = P.Model(dict(kind="oregonator", **synth.OREGONATOR))
    whole = u0.clone()
    P.rd_reaction_radau5(whole, model, 1e-3)
    part = u0.clone()
    cnt = torch.zeros((8, N), dtype=torch.int32, device="cuda")
    st = P.rd_stats()
    P.rd_reaction_radau5_cells(part[:, a:b], model, 1e-3, stats=st, cell_counters=cnt[:, a:b])
    torch.cuda.synchronize()
    assert st.n_cells == b - a and st.n_failed == 0
    assert torch.equal(part[:, a:b], whole[:, a:b])
    assert torch.equal(part[:, :a], u0[:, :a]) and torch.equal(part[:, b:], u0[:, b:])
    assert (cnt[1, a:b] >= 1).all() and (cnt[:, :a] == 0).all() and (cnt[:, b:] == 0).all()
