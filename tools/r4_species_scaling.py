"""Rock4 on the cfg-3 grid after one Strang step + adapt with 1, 2, 3 diffusing species (the others at
eps = 0): the per-round cost split into a fixed part and a per-species part."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
w = synth.cfg3()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
g.strang_step(P.Model(dict(w.model, m=w.m)), w.eps_diff, w.dt)
g.adapt()
_, u0 = g.leaf_tensors(); u0 = u0.clone()
for eps in ([w.eps_diff[0], 0, 0], [w.eps_diff[0], w.eps_diff[0], 0], [w.eps_diff[0]] * 3, list(w.eps_diff)):
    for k in range(3):
        g.set_values(u0)
        st = P.rd_stats()
        g.diffusion_rock4(eps, w.dt, stats=st)
        torch.cuda.synchronize()
    print(eps, f"kernel {st.rock4_kernel_ms:.3f} ms rounds {st.rock4_rounds} -> {1e3*st.rock4_kernel_ms/st.rock4_rounds:.2f} us/round", flush=True)
