"""Runs rd_reaction_radau5 once on BJ configs[1] (or a prefix of it) — for ncu captures."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1506_04651_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 22)
w = synth.cfg2()
u = torch.tensor(w.u[:, :n].copy(), device="cuda")
P.rd_reaction_radau5(u, P.Model(w.model), w.dt)
torch.cuda.synchronize()
print("ok", n)
