"""Small smooth test fields and leaf geometry helpers (test code)."""
import numpy as np

from tests.mr_ref import morton_decode


def front_field(dim, J, m=1, cx=0.4):
    n = 1 << J
    x = (np.arange(n) + 0.5) / n
    g = np.meshgrid(*([x] * dim), indexing="ij")
    if dim == 2:
        yy, xx = g
        r = np.hypot(xx - cx, yy - 0.55)
    else:
        zz, yy, xx = g
        r = np.sqrt((xx - cx) ** 2 + (yy - 0.55) ** 2 + (zz - 0.5) ** 2)
    comps = [np.tanh((0.25 - r) / 0.03), np.cos(6 * xx) * yy + 1.0, 0.5 + 0 * xx]
    k = 3
    while len(comps) < m:  # more species: fronts of other radii / widths
        comps.append(np.tanh((0.1 + 0.04 * k - r) / (0.02 + 0.01 * k)))
        k += 1
    return np.stack(comps[:m])


def leaf_geometry(dim, keys):
    lv = np.array([int(k) >> 58 for k in keys])
    cen = np.array([[(c + 0.5) * 2.0 ** -j for c in morton_decode(dim, int(k))[1]] for k, j in zip(keys, lv)])
    return lv, cen, 2.0 ** (-dim * lv)
