"""Single-core CPU oracle per phase (SURVEY §8(d) timing (a)): R (Radau5 per cell), D
(Rock4 per species) and A (mr_adapt) timed separately with ONE host thread on bounded samples of the BJ
configurations.  Writes one JSON object (stdout).  A reported baseline, not a target.

    python tools/oracle_1core.py [--budget SECONDS]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=20.0)
    a = ap.parse_args()
    out = {"threads": 1, "cpu": None, "phases": {}}
    try:
        with open("/proc/cpuinfo") as f:
            out["cpu"] = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        pass
    # R: cfg 2 cells (T = 1e-2) and cfg 4 leaves (T = dt/2), first n cells, one thread
    w2 = synth.cfg2()
    for name, u, model, T in (("R_cfg2", w2.u, oracle.Model(w2.model), w2.dt),):
        n = 2048
        t0 = time.perf_counter()
        oracle.radau5(u[:, :n].copy(), model, T, nthreads=1)
        dt = time.perf_counter() - t0
        out["phases"][name] = {"cells_per_s_core": n / dt, "sample": f"first {n} cells, T = {T}"}
    for cfg in (3, 4):
        w = synth.CONFIGS[cfg]()
        g = oracle.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, w.u.reshape(w.m, -1))
        model = oracle.Model(dict(w.model, m=w.m))
        nl = g.n_leaves
        _, u = g.leaves()
        n = min(nl, 4096)
        idx = np.linspace(0, nl - 1, n).astype(np.int64)  # evenly strided over the Morton leaf order
        t0 = time.perf_counter()
        oracle.radau5(np.ascontiguousarray(u[:, idx]), model, 0.5 * w.dt, nthreads=1)
        tr = time.perf_counter() - t0
        t0 = time.perf_counter()
        g.diffuse(w.eps_diff, w.dt, nthreads=1)
        td = time.perf_counter() - t0
        t0 = time.perf_counter()
        g.adapt()
        ta = time.perf_counter() - t0
        out["phases"][f"cfg{cfg}"] = {
            "leaves": nl,
            "R_cells_per_s_core": n / tr, "R_sample": f"{n} leaves evenly strided over the leaf order, one half step T = dt/2",
            "D_leaf_updates_per_s_core": nl / td, "D_sample": "one full D_dt over all leaves and species",
            "A_leaves_per_s_core": nl / ta, "A_sample": "one mr_adapt after the diffusion",
            "seconds": {"R": tr, "D": td, "A": ta}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
