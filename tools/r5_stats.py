"""Radau5 / Rock4 work statistics of the first Strang steps of a config (per-step counter totals)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = synth.CONFIGS[c]()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
model = P.Model(dict(w.model, m=w.m))
for it in range(nsteps):
    st = P.rd_stats()
    g.strang_step(model, w.eps_diff, w.dt, stats=st)
    d = st.as_dict()
    n = max(d.get("n_cells", 1), 1)
    print(f"step {it}: leaves {g.n_leaves} " + " ".join(f"{k}={v}" for k, v in d.items()), flush=True)
    print(f"   per cell-substep: attempts {d['n_attempts']/n:.2f} accept {d['n_accept']/n:.2f} reject {d['n_reject']/n:.2f} "
          f"newton {d['n_newton']/n:.2f} lu {d['n_lu']/n:.2f} jac {d['n_jac']/n:.2f} f {d['n_f']/n:.2f}", flush=True)
    g.adapt()
