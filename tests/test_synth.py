"""Seeded input generators (synth/): splitmix64 pinned to its published test
vector; recipes produce the shapes/ranges of SURVEY §8(d)."""
import numpy as np

import synth


def test_splitmix64_reference_vector():
    # splitmix64 (Steele, Lea, Flood 2014; Vigna's reference splitmix64.c), seed 0
    r = synth.SplitMix64(0)
    assert [r.next_u64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_block_equals_scalar_draws():
    a = synth.SplitMix64(7)
    b = synth.SplitMix64(7)
    blk = a.uniform_block(100)
    sc = np.array([b.uniform() for _ in range(100)])
    assert np.array_equal(blk, sc)
    assert a.state == b.state


def test_cfg1_shape_and_ranges():
    w = synth.cfg1()
    assert w.u.shape == (3, 128, 128)
    a, b, c = w.u
    assert 0.05 <= b.min() and b.max() <= 0.8 and 0.05 <= c.min() and c.max() <= 0.5
    assert np.allclose(a, 1.6 * c / (2e-3 + b))


def test_cfg2_cells():
    w = synth.cfg2(1 << 12)
    assert w.u.shape == (3, 4096)
    assert 0 <= w.u[1].min() and w.u[1].max() < 1


def test_cfg5_network():
    w = synth.cfg5(J=4)
    reac, prod, rate = w.model["reactants"], w.model["products"], w.model["rate"]
    assert reac.shape == (40, 2) and prod.shape == (40, 2)
    assert rate.min() >= 1e-2 and rate.max() <= 1e6
    for r in range(40):
        rs = set(int(x) for x in reac[r] if x >= 0)
        assert all(int(p) not in rs for p in prod[r] if p >= 0)
        nr = sum(1 for x in reac[r] if x >= 0)
        npr = sum(1 for x in prod[r] if x >= 0)
        assert npr <= nr  # species count never increases
    assert all(1e-4 <= e <= 5e-3 for e in w.eps_diff)
    assert w.u.min() > 0
