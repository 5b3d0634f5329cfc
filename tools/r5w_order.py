"""Warp-kernel Radau5 on the cfg-5 field (first half step): per-cell cost spread and what a longest-first
order (by the cells' own attempt counts: the ideal order) would save."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1506_04651_b200 as P
w = synth.cfg5()
u0 = torch.tensor(w.u.reshape(20, -1).copy(), device="cuda")
n = u0.shape[1]
model = P.Model(dict(w.model, m=20))
cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")


def timed(order, cnt=None):
    u = u0.clone()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    e[0].record(); P.rd_reaction_radau5_cells(u, model, 0.5 * w.dt, order=order, cell_counters=cnt); e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1])


for rep in range(2):
    print(f"none: {timed(None, cnt):.2f} ms")
c = cnt.cpu().numpy()
for q, name in ((0, "attempts"), (6, "newton"), (5, "lu")):
    print(f"{name}: mean {c[q].mean():.1f} p50 {np.percentile(c[q],50):.0f} p99 {np.percentile(c[q],99):.0f} max {c[q].max()}")
own = torch.argsort(cnt[6], descending=True, stable=True).to(torch.int32)
print(f"own (newton-descending): {timed(own):.2f} ms")
rs = np.random.RandomState(0)
print(f"random: {timed(torch.tensor(rs.permutation(n).astype(np.int32), device='cuda')):.2f} ms")
