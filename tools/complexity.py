"""SURVEY §8(f) N3 / paper experiment X2: per-node Radau5 complexity of one reaction half
step R_{dt/2} on a uniform 1024^2 BZ grid, from the library's per-cell counters.

complexity = right-hand-side evaluations + 3 per analytic Jacobian ("the Jacobian is computed
analytically involving three right-hand side evaluations").  Reports the histogram, the share of nodes
and the share of reaction work (sum of complexity) below 17 (the paper's threshold for BZ),
and writes the JSON to the path given (default gpurun_out/complexity_bz1024.json; the committed copy
lives in profiles/).  Initial data: the cfg-3 spiral fronts at level 10
(synthetic; the paper's data are not printed), dt = 1e-3, tol 1e-8."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_1506_04651_b200 as P

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/complexity_bz1024.json"
w = synth.cfg3()
u = torch.tensor(w.u.reshape(3, -1), device="cuda")  # row-major cells: complexity is per cell
n = u.shape[1]
cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")
st = P.rd_stats()
P.rd_reaction_radau5(u, P.Model(w.model), 0.5 * w.dt, stats=st, cell_counters=cnt)
c = cnt.cpu().numpy().astype(np.int64)
cplx = c[3] + 3 * c[4]
hist = np.bincount(cplx)
thr = 17
out = {
    "grid": "uniform 1024^2 (cfg-3 initial fronts), BZ q = 2e-3, one R_{dt/2}, dt = 1e-3, tol 1e-8",
    "complexity": "n_f + 3 n_jac per node (P:505-506)",
    "nodes": int(n),
    "min": int(cplx.min()), "median": float(np.median(cplx)), "max": int(cplx.max()),
    "share_nodes_below_17": float((cplx < thr).mean()),
    "share_work_below_17": float(cplx[cplx < thr].sum() / cplx.sum()),
    "paper_bz_share_work_below_17": 0.87,
    "histogram": {int(k): int(v) for k, v in enumerate(hist) if v},
    "reaction_ms": st.reaction_ms,
}
os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "histogram"}))
