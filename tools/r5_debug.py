"""Finds Radau5 cells that fail on the GPU (cfg 2) and reports them against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
import paper_1506_04651_b200 as P
w = synth.cfg2()
u = torch.tensor(w.u, device="cuda")
cnt = torch.zeros((8, u.shape[1]), dtype=torch.int32, device="cuda")
st = P.rd_stats()
rc = P.rd_reaction_radau5(u, P.Model(w.model), w.dt, stats=st, cell_counters=cnt, allow_stiff=True)
c = cnt.cpu().numpy()
bad = np.nonzero(c[7])[0]
print("rc", rc, "failed", st.n_failed, "idx", bad[:20], "status", c[7][bad[:20]])
for i in bad[:5]:
    print(i, w.u[:, i], dict(zip(P.COUNTER_NAMES, c[:, i])))
    o, oc, ost = oracle.radau5(w.u[:, i:i+1], oracle.Model(w.model), w.dt)
    print("  oracle", ost, dict(zip(oracle.COUNTER_NAMES, oc[:, 0])), o[:, 0], u[:, i].cpu().numpy())
