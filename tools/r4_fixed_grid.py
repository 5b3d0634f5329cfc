"""Rock4 on the cfg-3 grid after one Strang step + adapt (same grid for every variant), 3 calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
w = synth.cfg3()
u = torch.tensor(w.u.reshape(3, -1), device="cuda")
g = P.Grid.build(2, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(2, w.level_max, u))
_, u0 = g.leaf_tensors()
for k in range(3):
    g.set_values(u0)
    st = P.rd_stats()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(); g.diffusion_rock4(w.eps_diff, w.dt, stats=st); e[1].record(); torch.cuda.synchronize()
    print(f"D {e[0].elapsed_time(e[1]):.2f} ms rounds {st.rock4_rounds} -> {1e3*e[0].elapsed_time(e[1])/st.rock4_rounds:.1f} us/round", flush=True)
