"""Warp-per-cell Radau5 (m = 20) on the cfg-5 initial field: time and counters per half step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1506_04651_b200 as P
w = synth.cfg5()
u0 = torch.tensor(w.u.reshape(20, -1), device="cuda")
model = P.Model(dict(w.model, m=20))
n = u0.shape[1]
cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")
for rep in range(3):
    x = u0.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); P.rd_reaction_radau5(x, model, 0.5 * w.dt, cell_counters=cnt); ev[1].record(); torch.cuda.synchronize()
    c = cnt.cpu().numpy().astype(np.int64)
    print(f"n={n} ms={ev[0].elapsed_time(ev[1]):.3f} per-cell mean: " +
          " ".join(f"{k}={c[i].mean():.2f}" for i, k in enumerate(P.COUNTER_NAMES[:7])), flush=True)
