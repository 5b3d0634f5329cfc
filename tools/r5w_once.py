"""One warp-kernel Radau5 call on the first n cfg-5 cells (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
w = synth.cfg5()
u = torch.tensor(w.u.reshape(20, -1)[:, :n].copy(), device="cuda")
P.rd_reaction_radau5(u, P.Model(dict(w.model, m=20)), 0.5 * w.dt)
torch.cuda.synchronize()
print("ok", n)
