"""Times Strang steps + mr_adapt on a config with the adapt section profiler (RDMR_ADAPT_PROFILE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = synth.CONFIGS[c]()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
model = P.Model(dict(w.model, m=w.m))
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.strang_step(model, w.eps_diff, w.dt)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    g.adapt()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step {it}: strang {1e3*(t1-t0):.2f} ms adapt {1e3*(t2-t1):.2f} ms leaves {g.n_leaves}", flush=True)
