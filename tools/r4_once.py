"""One rd_diffusion_rock4 call on a config's initial grid (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = synth.CONFIGS[c]()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
st = P.rd_stats()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    g.diffusion_rock4(w.eps_diff, w.dt, stats=st)
    ev[1].record()
    torch.cuda.synchronize()
    print("rock4 ms", ev[0].elapsed_time(ev[1]))
print("rounds", st.rock4_rounds, "steps", st.rock4_steps, "rejects", st.rock4_rejects, "matvecs", st.rock4_matvecs, "s", st.rock4_s_min, st.rock4_s_max)
