"""Warp-kernel Radau5 on the first n cfg-5 cells: time (CUDA events) and work counters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_1506_04651_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
w = synth.cfg5()
u0 = torch.tensor(w.u.reshape(20, -1)[:, :n].copy(), device="cuda")
model = P.Model(dict(w.model, m=20))
for rep in range(2):
    u = u0.clone()
    st = P.rd_stats()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(); P.rd_reaction_radau5(u, model, 0.5 * w.dt, stats=st); e[1].record(); torch.cuda.synchronize()
    d = st.as_dict()
    print(f"{e[0].elapsed_time(e[1]):.1f} ms  att {d['n_attempts']} newt {d['n_newton']} lu {d['n_lu']} jac {d['n_jac']} f {d['n_f']} rej {d['n_reject']}")
