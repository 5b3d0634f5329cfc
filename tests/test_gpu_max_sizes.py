"""The level caps of include/rdmr.h (J = 14 in 2-D, J = 9 in 3-D: 2.7e8 / 1.3e8 finest cells) on the GPU,
checked through properties that hold at any size (the oracle would need minutes per case): the leaves
tile the domain exactly (sum of 2^{d(J-l)} = 2^{dJ}), keys are strictly increasing with levels in
[L_min, J], the grading invariant holds (face neighbours differ by at most one level), adaptation
keeps all of this, and a diffusion substep conserves mass (Neumann)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1506_04651_b200 as P
    P.lib()
    return P


def _front(dim, J):
    """tanh front of radius 0.3 and width 4 h_J around the centre (so the finest level is needed),
    row-major (x fastest), built on the device."""
    import torch
    n = 1 << J
    x = (torch.arange(n, device="cuda", dtype=torch.float64) + 0.5) / n
    if dim == 2:
        r2 = (x[None, :] - 0.45) ** 2 + (x[:, None] - 0.55) ** 2
    else:
        r2 = (x[None, None, :] - 0.45) ** 2 + (x[None, :, None] - 0.55) ** 2 + (x[:, None, None] - 0.5) ** 2
    return torch.tanh((0.3 - torch.sqrt(r2)) * (n / 4.0)).reshape(1, -1)


def _check_tiling(P, g, dim, lmin, J):
    keys, u = g.leaf_tensors()
    k = keys.cpu().numpy().view(np.uint64)
    lv = (k >> np.uint64(58)).astype(np.int64)
    assert (np.diff(k.astype(np.uint64)) > 0).all()
    assert lv.min() >= lmin and lv.max() <= J
    vol = (np.ones(len(lv), dtype=np.int64) << (dim * (J - lv))).sum()
    assert vol == 1 << (dim * J)
    return k, lv, u


def _graded(P, dim, k, lv, samples=20000):
    """Face neighbours of sampled leaves are leaves within one level (or refined by one level)."""
    key_of = {}
    rng = np.random.default_rng(0)
    idx = rng.choice(len(k), min(samples, len(k)), replace=False)
    leafset = set(int(x) for x in k)
    for i in idx:
        L, c = P.mr_key_decode(dim, int(k[i]))
        for a in range(dim):
            for s in (-1, 1):
                nb = list(c)
                nb[a] += s
                if nb[a] < 0 or nb[a] >= (1 << L):
                    continue
                # the neighbour region is covered by a leaf at level L-1, L or L+1 (graded tree)
                ok = P.mr_key_encode(dim, L, nb) in leafset
                if not ok and L > 0:
                    ok = P.mr_key_encode(dim, L - 1, [v >> 1 for v in nb]) in leafset
                if not ok:
                    ch = [2 * v + (1 if (a2 == a and s < 0) else 0) for a2, v in enumerate(nb)]
                    ok = P.mr_key_encode(dim, L + 1, ch) in leafset
                assert ok, (L, c, a, s)
                key_of[a] = True


@pytest.mark.parametrize("dim,lmin,J,eps", [(2, 6, 14, 1e-2), (3, 4, 9, 2e-3)])
def test_level_cap_build_adapt_diffuse(P, dim, lmin, J, eps):
    import torch
    u = P.mr_rowmajor_to_morton(dim, J, _front(dim, J))
    g = P.Grid.build(dim, lmin, J, eps, u)
    del u
    torch.cuda.empty_cache()
    k, lv, vals = _check_tiling(P, g, dim, lmin, J)
    assert lv.max() == J  # the front is resolved down to the finest level
    _graded(P, dim, k, lv)
    vol = np.ldexp(1.0, -dim * lv)
    m0 = (vals.cpu().numpy()[0] * vol).sum()
    g.diffusion_rock4([1e-4], 1e-6)
    _, v1 = g.leaf_tensors()
    assert abs((v1.cpu().numpy()[0] * vol).sum() - m0) <= 1e-12 * np.abs(vals.cpu().numpy()[0] * vol).sum()
    g.adapt()
    k2, lv2, _ = _check_tiling(P, g, dim, lmin, J)
    _graded(P, dim, k2, lv2)
