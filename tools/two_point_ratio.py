"""App. A "Ratio" analog (time with compact storage / time with the explicit-weight
matrix, Rock4 on the BZ problem in d = 2 and 3): the Rock4 kernel time of one D_{dt} on the cfg-3
(2-D, J = 10) and cfg-4 (3-D) grids after one Strang step + adapt, with RD_OP_TWO_POINT (explicit FP64
weights) and RD_OP_TWO_POINT_COMPACT (column + link type), the prediction operator for context.
Writes a JSON summary to argv[1] (default gpurun_out/two_point_ratio.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1506_04651_b200 as P  # noqa: E402
import synth  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/two_point_ratio.json"
reps = 5
res = {}
for c in (3, 4):
    w = synth.CONFIGS[c]()
    u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
    g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
    g.strang_step(P.Model(dict(w.model, m=w.m)), w.eps_diff, w.dt)
    g.adapt()
    _, u0 = g.leaf_tensors()
    u0 = u0.clone()
    row = {"n_leaves": g.n_leaves, "dim": w.dim, "J": w.level_max}
    for mode, name in ((0, "prediction"), (1, "two_point"), (2, "two_point_compact")):
        g.set_operator(mode)
        ks, rounds, mv, slots = [], 0, 0, 0
        for k in range(reps + 1):  # call 0 assembles the operator
            g.set_values(u0)
            st = P.rd_stats()
            g.diffusion_rock4(w.eps_diff, w.dt, stats=st)
            torch.cuda.synchronize()
            if k:
                ks.append(st.rock4_kernel_ms)
                rounds, mv, slots = st.rock4_rounds, st.rock4_matvecs, st.rock4_mat_slots
        ks.sort()
        med = ks[len(ks) // 2]
        row[name] = {"rock4_kernel_ms": med, "rounds": rounds, "matvecs": mv, "mat_slots": slots,
                     "us_per_round": 1e3 * med / max(rounds, 1), "all_ms": ks}
        print(c, name, row[name], flush=True)
    row["ratio_compact_over_explicit"] = row["two_point_compact"]["rock4_kernel_ms"] / row["two_point"]["rock4_kernel_ms"]
    res[f"cfg{c}"] = row
    print(c, "ratio", row["ratio_compact_over_explicit"], flush=True)
    del g
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
with open(out_path, "w") as f:
    json.dump(res, f, indent=1)
