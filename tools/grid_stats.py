"""Prints operator statistics of the MR configs after build and after one Strang step + adapt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
for c in (3, 4):
    w = synth.CONFIGS[c]()
    u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
    g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
    print(c, "build", g.stats())
    st = P.rd_stats()
    g.strang_step(P.Model(dict(w.model, m=3)), w.eps_diff, w.dt, stats=st)
    print(c, "rock4", st.rock4_steps, st.rock4_rejects, st.rock4_matvecs, st.rock4_s_min, st.rock4_s_max, st.rho1)
    g.adapt()
    print(c, "adapt", g.stats())
