"""Per-phase times and Rock4 rounds inside real Strang steps of a config (from the initial state)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = synth.CONFIGS[c]()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
model = P.Model(dict(w.model, m=w.m))
ev = lambda: torch.cuda.Event(enable_timing=True)
for it in range(nsteps):
    n, _, up = g.leaves()
    uu = g.leaf_tensors()[1]
    e = [ev() for _ in range(5)]
    st = P.rd_stats()
    e[0].record()
    P.rd_reaction_radau5(uu, model, 0.5 * w.dt)
    g.set_values(uu)
    e[1].record()
    g.diffusion_rock4(w.eps_diff, w.dt, stats=st)
    e[2].record()
    _, uu = g.leaf_tensors()
    P.rd_reaction_radau5(uu, model, 0.5 * w.dt)
    g.set_values(uu)
    e[3].record()
    if c in (3, 4):
        g.adapt()
    e[4].record()
    torch.cuda.synchronize()
    d = e[1].elapsed_time(e[2])
    print(f"step {it}: N={n} R1 {e[0].elapsed_time(e[1]):.2f} D {d:.2f} ms R2 {e[2].elapsed_time(e[3]):.2f} "
          f"A {e[3].elapsed_time(e[4]):.2f} | rock4 rounds {st.rock4_rounds} steps {st.rock4_steps} rejects "
          f"{st.rock4_rejects} s {st.rock4_s_min}-{st.rock4_s_max} -> {1e3 * d / max(st.rock4_rounds, 1):.1f} us/round",
          flush=True)
