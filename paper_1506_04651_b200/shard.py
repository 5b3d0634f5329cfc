"""Sharded Strang step: one MR problem stepped by P ranks, one process per GPU.

Decomposition of U_{n+1} = R_{dt/2} D_dt R_{dt/2} U_n and the re-adaptation:

* R (Radau5 per leaf): the leaves are independent.  Every rank computes the same cost keys
  (rd_reaction_cost) and the same cost-balanced contiguous intervals of the Morton leaf order
  (rd_shard_bounds; the paper's interval partition of the leaf set), integrates its
  own interval (rd_reaction_radau5_cells), and the intervals are all-gathered.
* D (Rock4 per species): eps_i A acts on species i alone, so species i is integrated on rank
  i mod P and broadcast from there.  No exchange inside a Rock4 step.
* A (mr_adapt): bit-exact for identical input, so each rank adapts its own replica of the tree with no
  exchange; all ranks keep identical grids (checked by the tests).

The tree and the leaf values are replicated (a BJ configuration uses well under 1 % of 180 GB), so this
divides the work of R and D, not the memory; the per-stage halo exchange of a row-sharded Rock4
 is the step after this one.  The collectives are torch.distributed (NCCL over NVLink on
GPUs, gloo in the CPU tests); every arithmetic step runs in the library's kernels.  The per-cell
arithmetic does not depend on the partition, so a sharded step equals the single-GPU step leaf by leaf
(R bit for bit; D bit for bit per species).
"""
from __future__ import annotations

from . import (RD_STRANG_DRD, RD_STRANG_RDR, Model, rd_reaction_cost, rd_reaction_radau5_cells,
               rd_shard_bounds)


class GridBackend:
    """The library on one GPU: a Grid, its model and options."""

    def __init__(self, grid, model: Model, ropts=None, kopts=None, balance=True):
        self.grid, self.model, self.ropts, self.kopts, self.balance = grid, model, ropts, kopts, balance

    def values(self):
        return self.grid.values_view()

    def commit(self, u):  # values() is a view of the grid's own memory
        pass

    def bounds(self, u, p):
        n = u.shape[1]
        cost = None
        if self.balance and p > 1 and n > 0 and self.model.m <= 4:
            cost = rd_reaction_cost(u, self.model, self.ropts)
        return rd_shard_bounds(n, cost, p)

    def react(self, u_part, T, stats=None):
        rd_reaction_radau5_cells(u_part, self.model, T, opts=self.ropts, stats=stats)

    def diffuse(self, eps, T, stats=None):
        self.grid.diffusion_rock4(eps, T, opts=self.kopts, stats=stats)

    def adapt(self):
        self.grid.adapt()


class ShardedStrang:
    """Strang steps of one problem over the ranks of `group` (default: the default process group, or a
    single rank when torch.distributed is not initialised)."""

    def __init__(self, backend, eps_diff, group=None):
        import torch.distributed as dist
        self.b, self.eps = backend, [float(e) for e in eps_diff]
        self.group = group
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.P = self.dist.get_world_size(group) if self.dist else 1
        self.last_bounds = None

    def _global(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def owner(self, i):
        """Rank that integrates species i in D."""
        return i % self.P

    def step(self, dt, scheme=RD_STRANG_RDR, stats=None):
        """stats: None or an rd_stats the backend's library calls add this rank's totals to."""
        if scheme == RD_STRANG_RDR:
            self.react(0.5 * dt, stats)
            self.diffuse(dt, stats)
            self.react(0.5 * dt, stats)
        elif scheme == RD_STRANG_DRD:
            self.diffuse(0.5 * dt, stats)
            self.react(dt, stats)
            self.diffuse(0.5 * dt, stats)
        else:
            raise ValueError(scheme)

    def adapt(self):
        self.b.adapt()

    def react(self, T, stats=None):
        u = self.b.values()
        bnd = self.b.bounds(u, self.P)
        self.last_bounds = bnd
        a, e = bnd[self.rank], bnd[self.rank + 1]
        if e > a:
            self.b.react(u[:, a:e], T, **({"stats": stats} if stats is not None else {}))
        self._gather_intervals(u, bnd)
        self.b.commit(u)

    def diffuse(self, T, stats=None):
        mine = [e if self.owner(i) == self.rank else 0.0 for i, e in enumerate(self.eps)]
        if any(e > 0.0 for e in mine):
            self.b.diffuse(mine, T, **({"stats": stats} if stats is not None else {}))
        if self.P > 1:
            u = self.b.values()
            for i, e in enumerate(self.eps):
                if e > 0.0:
                    row = u[i]  # contiguous species row of the SoA field
                    self._broadcast(row, self._global(self.owner(i)))
            self.b.commit(u)

    def _host_staged(self, t):
        """gloo has no CUDA all-gather: CUDA tensors travel through host memory there (NCCL moves them
        device to device).  Plumbing only, no arithmetic."""
        return t.is_cuda and self.dist.get_backend(self.group) == "gloo"

    def _broadcast(self, row, src):
        if self._host_staged(row):
            h = row.cpu()
            self.dist.broadcast(h, src=src, group=self.group)
            row.copy_(h)
        else:
            self.dist.broadcast(row, src=src, group=self.group)

    def _gather_intervals(self, u, bnd):
        """After R: every rank holds the whole field.  Intervals are padded to the longest one for the
        fixed-size all-gather, then copied into place."""
        if self.P == 1:
            return
        import torch
        m = u.shape[0]
        lens = [bnd[k + 1] - bnd[k] for k in range(self.P)]
        L = max(max(lens), 1)
        a = bnd[self.rank]
        send = torch.zeros((m, L), dtype=u.dtype, device=u.device)
        send[:, :lens[self.rank]] = u[:, a:a + lens[self.rank]]
        if self._host_staged(send):
            send = send.cpu()
        recv = [torch.empty_like(send) for _ in range(self.P)]
        self.dist.all_gather(recv, send, group=self.group)
        for k in range(self.P):
            if k != self.rank and lens[k]:
                u[:, bnd[k]:bnd[k + 1]] = recv[k][:, :lens[k]]
