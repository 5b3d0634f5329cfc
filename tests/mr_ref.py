"""Brute-force multiresolution reference for TINY grids (test code, independent
of oracle/src and of the product).

Dense per-level numpy arrays indexed by natural coordinates [k_x, k_y(, k_z)];
coarsening applies single collapses in a random sequential order (confluence
check, SURVEY §8(c) O.6 P7 / Appendix A probe 10), refinement/grading by plain
repeated sweeps.  Definitions followed: projection = mean of children
(P:559-563), prediction Eq. inter_1d tensor product, details and
level thresholds eps_j = 2^{(d/2)(j-J)} eps, graded tree
 with the radius-2 reading (DESIGN.md R-G2).
"""
from __future__ import annotations

import itertools

import numpy as np

R = 2  # grading radius (DESIGN.md R-G2)


def morton_key(dim, level, k):
    s = 0
    for b in range(level - 1, -1, -1):
        for a in range(dim):
            s = (s << 1) | ((k[a] >> b) & 1)
    return (level << 58) | s


class DenseTree:
    def __init__(self, dim, lmin, lmax, eps, m):
        self.dim, self.lmin, self.J, self.eps, self.m = dim, lmin, lmax, eps, m
        self.present = [np.zeros((1 << j,) * dim, dtype=bool) for j in range(lmax + 1)]
        self.leaf = [np.zeros((1 << j,) * dim, dtype=bool) for j in range(lmax + 1)]
        self.new = [np.zeros((1 << j,) * dim, dtype=bool) for j in range(lmax + 1)]
        self.u = [np.zeros((m,) + (1 << j,) * dim) for j in range(lmax + 1)]
        self.Q = [np.zeros((1 << j,) * dim) for j in range(lmax + 1)]

    # ---------------------------------------------------------------- helpers
    def cells(self, j):
        return itertools.product(range(1 << j), repeat=self.dim)

    def children(self, k):
        # Morton child order: digit (b_x, b_y[, b_z]) with x most significant
        for delta in range(1 << self.dim):
            yield tuple(2 * k[a] + ((delta >> (self.dim - 1 - a)) & 1) for a in range(self.dim))

    def project(self, j, k):
        ch = list(self.children(k))
        s = self.u[j + 1][(slice(None),) + ch[0]].copy()
        for c in ch[1:]:
            s = s + self.u[j + 1][(slice(None),) + c]
        self.u[j][(slice(None),) + tuple(k)] = s * (0.5 ** self.dim)

    def project_all(self):
        for j in range(self.J - 1, -1, -1):
            for k in self.cells(j):
                if self.present[j][k] and not self.leaf[j][k]:
                    self.project(j, k)

    def predict(self, j, k):
        """Value of (j, k) predicted from the parent's 3^d neighbourhood (mirrored)."""
        p = [x >> 1 for x in k]
        cb = [x & 1 for x in k]
        n = 1 << (j - 1)

        def val(o):
            idx = tuple(min(max(p[a] + o[a], 0), n - 1) for a in range(self.dim))
            assert self.present[j - 1][idx], "stencil node absent"
            return self.u[j - 1][(slice(None),) + idx]

        def step(um, u0, up, bit):
            t = 0.125 * (um - up)
            return u0 - t if bit else u0 + t

        if self.dim == 2:
            r = [step(val((-1, oy)), val((0, oy)), val((1, oy)), cb[0]) for oy in (-1, 0, 1)]
            return step(r[0], r[1], r[2], cb[1])
        q = []
        for oz in (-1, 0, 1):
            r = [step(val((-1, oy, oz)), val((0, oy, oz)), val((1, oy, oz)), cb[0]) for oy in (-1, 0, 1)]
            q.append(step(r[0], r[1], r[2], cb[1]))
        return step(q[0], q[1], q[2], cb[2])

    def significance(self):
        smax = np.ones(self.m)
        for j in range(self.J + 1):
            for i in range(self.m):
                vals = np.abs(self.u[j][i][self.leaf[j]])
                if vals.size:
                    smax[i] = max(smax[i], vals.max())
        for j in range(max(1, self.lmin), self.J + 1):
            for k in self.cells(j):
                if not self.present[j][k]:
                    continue
                d = self.u[j][(slice(None),) + k] - self.predict(j, k)
                t = d / smax
                self.Q[j][k] = np.max(t * t)

    def E(self, j):
        return np.ldexp(self.eps * self.eps, self.dim * (j - self.J))

    def inside(self, j, q):
        return all(0 <= x < (1 << j) for x in q)

    def box(self, center_lo, center_hi):
        return itertools.product(*[range(lo, hi + 1) for lo, hi in zip(center_lo, center_hi)])

    def collapsible(self, j, k):
        if j < self.lmin or j >= self.J or not self.present[j][k] or self.leaf[j][k]:
            return False
        for c in self.children(k):
            if not self.leaf[j + 1][c] or self.new[j + 1][c] or not (self.Q[j + 1][c] < self.E(j + 1)):
                return False
        lo = [2 * x - R for x in k]
        hi = [2 * x + 1 + R for x in k]
        for q in self.box(lo, hi):
            if self.inside(j + 1, q) and self.present[j + 1][q] and not self.leaf[j + 1][q]:
                return False
        return True

    def coarsen_random(self, rng):
        while True:
            cand = [(j, k) for j in range(self.J) for k in self.cells(j) if self.collapsible(j, k)]
            if not cand:
                return
            rng.shuffle(cand)
            for j, k in cand:
                if self.collapsible(j, k):
                    for c in self.children(k):
                        self.present[j + 1][c] = False
                        self.leaf[j + 1][c] = False
                    self.leaf[j][k] = True

    def refine(self, j, k):
        self.leaf[j][k] = False
        for c in self.children(k):
            self.present[j + 1][c] = True
            self.leaf[j + 1][c] = True
            self.new[j + 1][c] = True

    def grade(self):
        while True:
            todo = set()
            for j in range(self.J + 1):
                for k in self.cells(j):
                    if not self.present[j][k] or self.leaf[j][k]:
                        continue
                    for q in self.box([x - R for x in k], [x + R for x in k]):
                        if not self.inside(j, q) or self.present[j][q]:
                            continue
                        a, la = list(q), j
                        while True:
                            a = [x >> 1 for x in a]
                            la -= 1
                            if self.present[la][tuple(a)]:
                                todo.add((la, tuple(a)))
                                break
            if not todo:
                return
            for la, a in todo:
                if self.leaf[la][a]:
                    self.refine(la, a)

    # ---------------------------------------------------------------- public
    @classmethod
    def build(cls, dim, lmin, lmax, eps, u_rowmajor, seed=0):
        m = u_rowmajor.shape[0]
        t = cls(dim, lmin, lmax, eps, m)
        for j in range(lmax + 1):
            t.present[j][...] = True
        t.leaf[lmax][...] = True
        # row-major [m, (z,) y, x] -> [m, x, y(, z)]
        t.u[lmax] = np.ascontiguousarray(np.transpose(u_rowmajor, (0,) + tuple(range(dim, 0, -1))))
        t.project_all()
        t.significance()
        t.coarsen_random(np.random.default_rng(seed))
        return t

    def adapt(self, seed=0):
        self.project_all()
        self.significance()
        for j in range(self.J + 1):
            self.new[j][...] = False
        r0 = [(j, k) for j in range(self.J) for k in self.cells(j)
              if self.leaf[j][k] and self.Q[j][k] > self.E(j)]
        for j, k in r0:
            self.refine(j, k)
        self.grade()
        for j in range(1, self.J + 1):
            vals = {k: self.predict(j, k) for k in self.cells(j) if self.new[j][k]}
            for k, v in vals.items():
                self.u[j][(slice(None),) + k] = v
        self.coarsen_random(np.random.default_rng(seed))
        for j in range(self.J + 1):
            self.new[j][...] = False

    def leaves(self):
        out = []
        for j in range(self.J + 1):
            for k in self.cells(j):
                if self.leaf[j][k]:
                    out.append((morton_key(self.dim, j, k), self.u[j][(slice(None),) + k].copy()))
        out.sort(key=lambda t: t[0])
        keys = np.array([t[0] for t in out], dtype=np.uint64)
        vals = np.array([t[1] for t in out]).T.copy() if out else np.zeros((self.m, 0))
        return keys, vals


def morton_decode(dim, key):
    level = key >> 58
    s = key & ((1 << 58) - 1)
    k = [0] * dim
    for b in range(level):
        for a in range(dim - 1, -1, -1):
            k[a] |= (s & 1) << b
            s >>= 1
    return level, tuple(k)


def tree_from_leaves(dim, lmin, lmax, eps, keys, u):
    t = DenseTree(dim, lmin, lmax, eps, u.shape[0])
    for r, key in enumerate(keys):
        j, k = morton_decode(dim, int(key))
        t.present[j][k] = True
        t.leaf[j][k] = True
        t.u[j][(slice(None),) + k] = u[:, r]
        while j > 0:
            k = tuple(x >> 1 for x in k)
            j -= 1
            t.present[j][k] = True
    t.project_all()
    return t
