#!/usr/bin/env python
"""Benchmark of the B200 Strang / Radau5 / Rock4 / MR hot path (BASELINE.json metric:
leaf-cell updates/s per Strang step at 1 B200; % FP64 peak (Radau5), % HBM (Rock4)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One JSON line on rank 0.  Default: config 4 (BJ configs[3], the largest single-GPU configuration).
A "step" is one pass of the hot path over the config's synthetic input:
  config 2  one rd_reaction_radau5 over T = 1e-2 of 2^22 independent BZ cells (BJ configs[1]);
            unit = cells integrated
  config 1/5  one rd_strang_step on the uniform grid (BJ configs[0] / configs[4])
  config 3/4  one rd_strang_step + mr_adapt on the MR grid (BJ configs[2] / configs[3]), the paper's
            S = A + R + D per step
  Strang configs: the warm-up steps run on a throw-away grid, then the grid is rebuilt from the
  initial data and the K timed steps are the run's steps 1..K (BJ: 1 / 20 / 10 / 5 steps).
  unit for 1/3/4/5 = leaf cells at the start of the step
Multi-GPU (`--gpus N` is authoritative: re-executed under torch.distributed.run when no launcher set
WORLD_SIZE): the units are independent (north_star: independent cells / the same problem per rank),
every rank runs its own copy of the per-GPU workload with no data-path collective ("scaling": "weak").
`roofline` is the dominant phase's entry; `roofline.phases` has R (Radau5, FP64), D (Rock4, HBM) and A
(mr_adapt, HBM) with their shares of the step.
`--impl reference` times the CPU oracle (oracle/, plain scalar C++) on a bounded sample of the same
workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 34.2  # profiles/r01_fp64_peak.txt: DFMA-chain microbenchmark on this pool's B200 at 1965 MHz
CONFIG_NAMES = {1: "cfg1_bz_uniform_128x128", 2: "cfg2_radau5_batch_2^22", 3: "cfg3_bz_mr2d_J10",
                4: "cfg4_bz_mr3d_J7", 5: "cfg5_massaction20_uniform_512x512",
                6: "cfg6_nagumo_mr2d_J10_rk4"}  # 6: SURVEY §8(f) N1, not a BASELINE.json config


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4,
                    help="BJ configs[c-1]; default 4 = the largest single-GPU configuration (3-D MR, ~1.07e6 leaves)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="N > 1: step ONE problem over the N ranks (paper_1506_04651_b200/shard.py, strong scaling) "
                         "instead of one independent problem per rank (weak scaling, the default)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def ensure_world(a):
    """--gpus N is authoritative: without a launcher (no WORLD_SIZE) and N > 1 this process re-executes
    itself under torch.distributed.run with N ranks; under a launcher WORLD_SIZE must equal N."""
    if "WORLD_SIZE" not in os.environ:
        if a.gpus > 1:
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                       f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
                                       "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:])
        return
    world = int(os.environ["WORLD_SIZE"])
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        """Starts the sampler and waits (<= 3 s) for its first sample, so that a short timed region that
        follows is covered."""
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
            return
        t_end = time.time() + 3.0
        while time.time() < t_end and os.path.getsize(self.path) == 0:
            time.sleep(0.02)

    def stop(self, t0=None, t1=None):
        """Summary of the samples taken in the wall-clock window [t0, t1] (all samples if None)."""
        import datetime
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        rows = []
        with open(self.path) as f:
            for ln in f:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) >= 8:
                    try:
                        ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    except ValueError:
                        ts = None
                    if t0 is None or ts is None or (t0 - 0.05 <= ts <= t1 + 0.05):
                        rows.append(parts[1:])
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def measured_traffic(workload, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/*traffic.json), else None."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):
        try:
            with open(p) as f:
                v = json.load(f).get(workload, {}).get(kernel)
            if v is not None:
                best = v
        except (OSError, ValueError):
            pass
    return best


def flush_l2(buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


# ---------------------------------------------------------------------------------- workloads
def radau5_flops(cnt_tot, m, F, Jf):
    """Algorithmic FLOPs of Radau5 from the counters."""
    att, acc, rej, nf, njac, nlu, nnewt = cnt_tot
    return (nf * F + njac * Jf + nlu * (10 * m ** 3 / 3 + 3 * m ** 2) + nnewt * (10 * m ** 2 + 48 * m)
            + att * (2 * m ** 2 + 25 * m))


class Cfg2:
    """BJ configs[1]: 2^22 independent BZ cells, one Radau5 integration over T = 1e-2."""

    metric_unit = "cells/s"

    def __init__(self, P, torch, rank):
        import synth
        self.P, self.torch = P, torch
        w = synth.cfg2()
        self.w = w
        self.model = P.Model(w.model)
        self.T = w.dt
        self.n = w.u.shape[1]
        self.u0 = torch.tensor(w.u, device="cuda")
        self.u = torch.empty_like(self.u0)
        self.host_in = torch.tensor(w.u).pin_memory()
        self.host_out = torch.empty_like(self.host_in).pin_memory()
        self.launches_per_step = 1
        self.cnt = torch.zeros((8, self.n), dtype=torch.int32, device="cuda")

    def reset(self):
        self.u.copy_(self.u0)

    def units(self):
        return self.n

    def step(self, stats=None, timed=False):
        self.P.rd_reaction_radau5(self.u, self.model, self.T, stats=stats)

    def step_e2e(self):
        torch = self.torch
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        self.u.copy_(self.host_in, non_blocking=True)
        self.P.rd_reaction_radau5(self.u, self.model, self.T)
        self.host_out.copy_(self.u, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e), 8 * 3 * self.n, 8 * 3 * self.n, self.n

    def roofline(self, ms_kernel):
        st = self.P.rd_stats()
        self.reset()
        self.P.rd_reaction_radau5(self.u, self.model, self.T, stats=st, cell_counters=self.cnt)
        tot = self.cnt[:7].to(self.torch.int64).sum(dim=1).cpu().numpy()
        fl = radau5_flops(tot, 3, 14, 12)
        ach = fl / (ms_kernel * 1e-3) / 1e12
        return {"bound": "alu", "kernel": "radau5_thread<3>", "achieved": ach, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS, "traffic": None,
                "peak_source": "profiles/r01_fp64_peak.txt (measured DFMA chain, 1965 MHz)",
                "algorithmic_flop_per_launch": fl, "counters": dict(zip(
                    ("attempt", "accept", "reject", "f", "jac", "lu", "newton"), [int(x) for x in tot]))}

    def config(self):
        return workload_config(2)



class StrangCfg:
    """BJ configs[0] / [2] / [3] / [4]: Strang steps (RDR) on the (MR) grid; configs 3/4 re-adapt
    after every step.  A bench step = R(dt/2) + D(dt) + R(dt/2) [+ mr_adapt], timed per phase
    with CUDA events on the launching stream; the state advances from step to step (as in the run)."""

    metric_unit = "leaf-cell updates/s"

    def __init__(self, P, torch, rank, cfg):
        import synth
        self.P, self.torch, self.cfg = P, torch, cfg
        w = synth.CONFIGS[cfg]()
        self.w = w
        self.adaptive = cfg in (3, 4, 6)
        self.scheme = P.RD_STRANG_RDR | (P.RD_STRANG_RK4 if cfg == 6 else 0)  # NAGUMO: RK4 reactions (N1)
        self.model = P.Model(dict(w.model, m=w.m))
        self.u_init = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
        self.ropts, self.kopts = P.radau5_opts(), P.rock4_opts()
        self.phase_ms = {"R": 0.0, "D": 0.0, "A": 0.0}
        self.flops = 0.0
        self.r4_bytes = 0.0
        self.r4_kernel_ms = 0.0
        self.r4_kernel = "k_rock4"
        self.leaves_sum = 0
        self.mr_bytes = 0.0
        self.cnt = None
        self.kernels = {"R": 0, "D": 0, "A": 0}
        self.S = None
        self.restart()

    def enable_shard(self):
        """Sharded Strang step: R on cost-balanced leaf intervals, D on species i mod N,
        A replicated; Radau5 configurations only."""
        if self.cfg == 6:
            raise SystemExit("--shard: the RK4 (NAGUMO) configuration is not sharded")
        from paper_1506_04651_b200.shard import GridBackend, ShardedStrang
        self._shard_cls = (GridBackend, ShardedStrang)
        self.restart()

    def _advance(self, stats=None):
        if self.S is not None:
            self.S.step(self.w.dt, self.P.RD_STRANG_RDR, stats=stats)
        else:
            self.g.strang_step(self.model, self.w.eps_diff, self.w.dt, self.scheme, self.ropts, self.kopts,
                               stats=stats)

    def restart(self):
        """A fresh grid from the initial data (mr_grid_build): the timed steps are the run's first steps."""
        w, P = self.w, self.P
        um = P.mr_rowmajor_to_morton(w.dim, w.level_max, self.u_init)
        self.g = None
        self.g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, um)
        self.n_last = self.g.n_leaves
        self._n_internal = self.g.info()["n_internal"]
        if getattr(self, "_shard_cls", None):
            B, S = self._shard_cls
            self.S = S(B(self.g, self.model, self.ropts, self.kopts), w.eps_diff)

    def reset(self):
        pass

    def units(self):
        return self.g.n_leaves

    def step(self, stats=None, timed=False):
        """One Strang step through the public call rd_strang_step (RDR, longest-first cell order by the cost proxy in both
        reaction half steps; RK4 reactions for NAGUMO) + mr_adapt; the phase split comes from the library's
        own CUDA events (rd_stats.reaction_ms / diffusion_ms / rock4_kernel_ms), the adapt phase from
        events here."""
        torch = self.torch
        stream = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        n = self.g.n_leaves
        st = self.P.rd_stats()
        ev[0].record(stream)
        self._advance(stats=st)
        ev[1].record(stream)
        if self.adaptive:
            self.g.adapt()
        ev[2].record(stream)
        torch.cuda.synchronize()
        if timed and self.adaptive:
            # N_tree (24m + 24) B (projection, details, flags) + N_leaf (16m + 16) B
            # (compaction) per adaptation, on the tree it starts from
            m = self.w.m
            self.mr_bytes += (n + self._n_internal) * (24 * m + 24) + n * (16 * m + 16)
        if self.adaptive:
            self._n_internal = self.g.info()["n_internal"]
        if timed:
            self.phase_ms["R"] += st.reaction_ms
            self.phase_ms["D"] += st.diffusion_ms
            self.phase_ms["A"] += ev[1].elapsed_time(ev[2])
            tot = [st.n_attempts, st.n_accept, st.n_reject, st.n_f, st.n_jac, st.n_lu, st.n_newton]
            m = self.w.m
            F, Jf = (14, 12) if m == 3 else (190, 400)
            self.flops += radau5_flops(tot, m, F, Jf)
            self.r4_bytes += 24.0 * n * st.rock4_matvecs
            self.r4_kernel_ms += st.rock4_kernel_ms
            self.r4_kernel = "k_rock4_mat" if st.rock4_mat_slots > 0 else "k_rock4"
            self.kernels["R"] += 2
            self.kernels["D"] += 1
            self.leaves_sum += n
        return ev[0].elapsed_time(ev[2])

    def step_e2e(self):
        """Through the public API (rd_strang_step + mr_adapt) with the leaf state staged from / to pinned
        host buffers inside the timed region."""
        torch = self.torch
        host = self.g.values_view().cpu().pin_memory()
        w = self.w
        cap = w.m << (w.dim * w.level_max)  # leaves never exceed the finest level's cells
        if getattr(self, "_out_pinned", None) is None or self._out_pinned.numel() < cap:
            self._out_pinned = torch.empty(cap, dtype=torch.float64, pin_memory=True)  # outside the timed region
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        n = host.shape[1]
        self.g.values_view().copy_(host, non_blocking=True)  # H2D straight into the grid's leaf values
        self._advance()
        if self.adaptive:
            self.g.adapt()
        u2 = self.g.values_view()
        out = self._out_pinned[:u2.numel()].view(u2.shape)
        out.copy_(u2, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e), host.numel() * 8, out.numel() * 8, n

    def phase_rooflines(self, total_ms):
        """Each phase against its own roofline: R (Radau5 or RK4) on the FP64 pipe,
        D (Rock4 kernel, CUDA events around its launch) and A (mr_adapt) on HBM by algorithmic bytes."""
        ph = self.phase_ms
        hbm = peaks().get("hbm_gbs", 6553.9)
        share = {k: v / total_ms for k, v in ph.items()}
        out = {}
        if self.cfg == 6:  # NAGUMO: RK4 reactions, read + write the state in each of the two half steps
            byts = 2 * self.leaves_sum * 2 * 8 * self.w.m
            ach = byts / (ph["R"] * 1e-3) / 1e9
            out["R"] = {"bound": "hbm", "kernel": "k_rk4<1>", "achieved": ach, "peak": hbm, "unit": "GB/s",
                        "frac": ach / hbm, "traffic": None, "ms": ph["R"], "share": share["R"]}
        else:
            ach = self.flops / (ph["R"] * 1e-3) / 1e12
            out["R"] = {"bound": "alu", "kernel": "radau5_thread<3>" if self.w.m <= 4 else "radau5_warp<20>",
                        "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": ach / FP64_PEAK_TFLOPS,
                        "traffic": measured_traffic(CONFIG_NAMES[self.cfg], "radau5_thread<3>" if self.w.m <= 4
                                                    else "radau5_warp<20>"),
                        "peak_source": "profiles/r01_fp64_peak.txt (builder-measured DFMA chain, 1965 MHz; "
                                       "MEASURED_PEAKS.json has no FP64 entry)",
                        "algorithmic_flop": self.flops, "ms": ph["R"], "share": share["R"]}
        kms = self.r4_kernel_ms if self.r4_kernel_ms > 0 else ph["D"]
        ach = self.r4_bytes / (kms * 1e-3) / 1e9
        nlaunch = max(self.kernels["D"], 1)
        out["D"] = {"bound": "hbm", "kernel": self.r4_kernel, "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": measured_traffic(CONFIG_NAMES[self.cfg], self.r4_kernel),
                    "traffic_unit": "bytes per launch (ncu, profiles/*_traffic.json)",
                    "algorithmic_bytes_per_launch": self.r4_bytes / nlaunch, "kernel_ms_per_launch": kms / nlaunch,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)", "ms": ph["D"], "share": share["D"],
                    "note": "24 B per leaf per species per stage (SURVEY §8(d)) / kernel time from CUDA events "
                            "around the Rock4 launch (operator assembly is in phase D, not in the kernel time)"}
        if self.adaptive and ph["A"] > 0:
            ach = self.mr_bytes / (ph["A"] * 1e-3) / 1e9
            out["A"] = {"bound": "hbm", "kernel": "mr_adapt (all kernels of the call)", "achieved": ach, "peak": hbm,
                        "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                        "algorithmic_bytes": self.mr_bytes, "ms": ph["A"], "share": share["A"],
                        "note": "SURVEY §8(d): N_tree (24m + 24) + N_leaf (16m + 16) B per adaptation / the "
                                "call's CUDA-event time"}
        return out

    def roofline(self, total_ms):
        """The dominant phase's roofline, with every phase's under 'phases'."""
        phases = self.phase_rooflines(total_ms)
        dom = max(phases, key=lambda k: self.phase_ms[k])
        r = dict(phases[dom])
        r["phase"] = dom
        r["phases"] = phases
        r["phase_ms"] = self.phase_ms
        return r

    def config(self):
        return workload_config(self.cfg)


WORKLOADS = {1: lambda P, t, r: StrangCfg(P, t, r, 1), 2: Cfg2, 3: lambda P, t, r: StrangCfg(P, t, r, 3),
             4: lambda P, t, r: StrangCfg(P, t, r, 4), 5: lambda P, t, r: StrangCfg(P, t, r, 5),
             6: lambda P, t, r: StrangCfg(P, t, r, 6)}


def run_ours(a):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_1506_04651_b200 as P
    P.lib()
    W = WORKLOADS[a.config](P, torch, rank)
    shard = bool(a.shard) and world > 1
    if shard:
        if not hasattr(W, "enable_shard"):
            raise SystemExit("--shard applies to the Strang configurations")
        W.enable_shard()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda").view(torch.float64)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        W.reset()
        W.step()
    torch.cuda.synchronize()
    if hasattr(W, "restart"):  # warm-up ran on a throw-away grid; time the run's first steps
        # one untimed step on a first fresh grid: the first adaptation of a fresh grid while the warm-up
        # grid's blocks are fragmented in the stream-ordered pool grows the pool (~80 ms once on cfg 4,
        # tools/first_step.py); the timed grid then finds its buffers in the pool
        W.restart()
        W.step()
        torch.cuda.synchronize()
        W.restart()
        torch.cuda.synchronize()
        W.n0 = W.g.n_leaves  # reported as leaves_at_start (top level; not a workload key)
    clocks = Clocks(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    units = 0
    barrier()
    launches0 = P.kernel_launches()
    t_wall0 = time.time()
    inner = []
    for k in range(a.steps):
        W.reset()
        flush_l2(flush)
        units += W.units()
        ev[k][0].record(stream)
        inner.append(W.step(timed=True))  # device time of the step's own work (CUDA events), or None
        ev[k][1].record(stream)
    barrier()
    launches = P.kernel_launches() - launches0
    t_wall1 = time.time()
    # a timed region shorter than the sampler's 100 ms period is followed by untimed steps of the same
    # workload (not in any reported number) so that the clocks under this load are sampled
    while time.time() - t_wall0 < 0.35:
        W.reset()
        W.step()
        torch.cuda.synchronize()
    ck = clocks.stop(t_wall0, max(t_wall1, time.time()))
    if ck is not None:
        ck["window_s"] = round(max(t_wall1, time.time()) - t_wall0, 3)
        ck["timed_s"] = round(t_wall1 - t_wall0, 3)
    # a Strang step returns the CUDA-event time from its first launch to the end of mr_adapt; the outer
    # events would also count the host's bookkeeping after the step's final synchronisation
    ms = [t if t is not None else s.elapsed_time(e) for t, (s, e) in zip(inner, ev)]
    total_ms = float(np.sum(ms))
    # e2e through the public API with pinned host buffers, copies inside the timed region
    e2e = []
    if hasattr(W, "restart"):  # e2e over the same first steps of the run
        W.restart()
        torch.cuda.synchronize()
    for k in range(a.steps):  # the same steps as the device-timed window
        W.reset()
        flush_l2(flush)
        torch.cuda.synchronize()
        e2e.append(W.step_e2e())
    e2e_ms = float(np.sum([x[0] for x in e2e]))
    e2e_units = float(np.sum([x[3] for x in e2e]))
    total_ms, e2e_ms = max_over_ranks([total_ms, e2e_ms], world, device="cuda")
    roof = W.roofline(total_ms if hasattr(W, "phase_ms") else float(np.median(ms)))
    out = None
    if rank == 0:
        jobs = 1 if shard else world  # sharded: the ranks step ONE problem
        value = aggregate_value(units, total_ms, jobs)
        e2e_val = aggregate_value(e2e_units, e2e_ms, jobs)
        cpu = None
        if not a.no_cpu_baseline:
            import oracle
            cpu = oracle_rate(a.config, oracle, max_steps=1 if a.config != 2 else 3, budget_s=30.0)
        out = {"metric": "leaf-cell updates/s per Strang step" if a.config != 2 else
               "cells integrated/s (Radau5 reaction substep, T=1e-2)",
               "value": value, "unit": W.metric_unit, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
               "ms_per_step": total_ms / a.steps, "higher_is_better": True, "scaling": "strong" if shard else "weak",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64, SURVEY §8(d) recipe)",
               "config": dict(W.config(), parallelism=(f"shard{world}" if shard else f"replicas{world}")),
               "clocks": ck,
               "e2e": {"value": e2e_val, "unit": W.metric_unit, "h2d_bytes_per_step": int(e2e[-1][1]),
                       "d2h_bytes_per_step": int(e2e[-1][2])},
               "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "impl": "ours",
               "step_ms": [round(x, 4) for x in ms]}
        if hasattr(W, "n0"):
            out["leaves_at_start"] = W.n0
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return out


def max_over_ranks(values, world, device="cpu"):
    """Device-timed durations -> their maximum over ranks (the job's time; B200 timing rule).  Units
    are independent per rank (weak scaling, no data-path collective): value = units * world / max_t."""
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def aggregate_value(units_per_rank, max_ms, world):
    return units_per_rank * world / (max_ms * 1e-3)


def oracle_rate(cfg, orc, max_steps=3, budget_s=90.0, warmup=0):
    """The CPU oracle (oracle/, plain scalar C++, threaded over independent cells / species) timed on
    a bounded sample of config `cfg` on this host's cores.  cfg 2: the first 32 768 cells per step;
    Strang configs: consecutive oracle Strang steps (+ mr_adapt for 3/4) from the initial state, until
    max_steps or budget_s is reached (at least one)."""
    import synth
    nthr = os.cpu_count() or 1
    w = synth.CONFIGS[cfg]()
    if cfg == 2:
        ncells = 32768
        model = orc.Model(w.model)
        vals = []
        for k in range(warmup + max_steps):
            u = w.u[:, :ncells].copy()
            t0 = time.perf_counter()
            orc.radau5(u, model, w.dt, nthreads=nthr)
            if k >= warmup:
                vals.append(ncells / (time.perf_counter() - t0))
        return {"value": float(np.mean(vals)), "unit": "cells/s", "cores": nthr, "kind": "oracle",
                "ms_per_step": 1e3 * ncells / float(np.mean(vals)),
                "sample": f"first {ncells} of the 2^22 cfg-2 cells per step, {len(vals)} step(s), threaded oracle"}
    adaptive = cfg in (3, 4, 6)
    scheme = orc.STRANG_RK4 if cfg == 6 else 0
    o = orc.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, w.u.reshape(w.m, -1))
    model = orc.Model(dict(w.model, m=w.m))
    units, secs, n = 0, 0.0, 0
    t_start = time.perf_counter()
    while n < max_steps + warmup:
        nl = o.n_leaves
        t0 = time.perf_counter()
        o.strang(model, w.eps_diff, w.dt, scheme, nthreads=nthr)
        if adaptive:
            o.adapt()
        dt = time.perf_counter() - t0
        if n >= warmup:
            units += nl
            secs += dt
        n += 1
        if time.perf_counter() - t_start > budget_s and n > warmup:
            break
    return {"value": units / secs, "unit": "leaf-cell updates/s", "cores": nthr, "kind": "oracle",
            "ms_per_step": 1e3 * secs / max(1, n - warmup),
            "sample": f"{n - warmup} consecutive Strang step(s){' + mr_adapt' if adaptive else ''} of "
                      f"{CONFIG_NAMES[cfg]} from its initial state (time-bounded), threaded oracle"}


L2_NOTE = "flushed between timed steps (256 MiB write)"


def workload_config(cfg):
    """`config` of the JSON line: the workload only, identical in both arms (built on the host)."""
    import synth
    w = synth.CONFIGS[cfg]()
    if cfg == 2:
        return {"workload": CONFIG_NAMES[2], "cells": int(w.u.reshape(w.m, -1).shape[1]), "m": w.m, "T": w.dt,
                "tol": 1e-8, "l2": L2_NOTE}
    return {"workload": CONFIG_NAMES[cfg], "dim": w.dim, "J": w.level_max, "L_min": w.level_min,
            "eps_mr": w.eps_mr, "m": w.m, "dt": w.dt, "scheme": "RDR", "adapt_each_step": cfg in (3, 4, 6),
            "tol": 1e-8, "l2": L2_NOTE}


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on the host cores, rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    import oracle
    oracle.lib()
    cpu = oracle_rate(a.config, oracle, max_steps=a.steps, budget_s=150.0, warmup=min(a.warmup, 1))
    v = cpu["value"]
    out = {"metric": "leaf-cell updates/s per Strang step" if a.config != 2 else
           "cells integrated/s (Radau5 reaction substep, T=1e-2)", "value": v, "unit": cpu["unit"],
           "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": cpu.get("ms_per_step"),
           "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64)",
           "config": dict(workload_config(a.config), parallelism=f"replicas{world}"), "impl": "reference",
           "l2_note": "the oracle arm runs on the host: L2 flushing does not apply", "cpu_baseline": cpu,
           "e2e": {"value": v, "unit": cpu["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    args = parse()
    ensure_world(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
