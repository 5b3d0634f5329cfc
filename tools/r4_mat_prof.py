"""Rock4 on the cfg-3 (or cfg-4) grid after one Strang step + adapt: first call after the adapt
(includes the operator assembly) vs repeated calls on the same grid, us per round."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = synth.CONFIGS[c]()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
spec = dict(w.model, m=w.m)
g.strang_step(P.Model(spec), w.eps_diff, w.dt)
for rep in range(2):
    g.adapt()
    _, u0 = g.leaf_tensors()
    u0 = u0.clone()
    for k in range(3):
        g.set_values(u0)
        st = P.rd_stats()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(); g.diffusion_rock4(w.eps_diff, w.dt, stats=st); e[1].record(); torch.cuda.synchronize()
        t = e[0].elapsed_time(e[1])
        print(f"adapt {rep} call {k}: D {t:.3f} ms rounds {st.rock4_rounds} -> {1e3*t/st.rock4_rounds:.2f} us/round"
              f" slots {st.rock4_mat_slots} N {g.n_leaves}", flush=True)
