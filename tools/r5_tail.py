"""Radau5 on the leaves of the cfg-3 grid (T = dt/2): time, counters, and the per-cell cost spread."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1506_04651_b200 as P
w = synth.cfg3()
u = torch.tensor(w.u.reshape(3, -1), device="cuda")
g = P.Grid.build(2, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(2, w.level_max, u))
model = P.Model(dict(w.model, m=3))
_, uu = g.leaf_tensors()
n = uu.shape[1]
cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")
for rep in range(3):
    x = uu.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); P.rd_reaction_radau5(x, model, 0.5 * w.dt, cell_counters=cnt); ev[1].record(); torch.cuda.synchronize()
    c = cnt.cpu().numpy()
    print(f"n={n} ms={ev[0].elapsed_time(ev[1]):.3f} attempts={c[0].sum()} newton={c[6].sum()} "
          f"att/cell mean={c[0].mean():.1f} max={c[0].max()} p99={np.percentile(c[0],99):.0f}")
# cost of the same cells sorted by descending attempts (LPT order) for comparison
order = torch.tensor(np.argsort(-c[0], kind="stable"), device="cuda")
xs = uu[:, order].contiguous()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(); P.rd_reaction_radau5(xs, model, 0.5 * w.dt); ev[1].record(); torch.cuda.synchronize()
print(f"LPT-ordered ms={ev[0].elapsed_time(ev[1]):.3f}")
