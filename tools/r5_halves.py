"""The two reaction half steps of one RDR Strang step on a config's initial grid, piecewise through
the public calls: time and work of each half, and how much of the second half's time is its LPT order
(the first half's attempt counts) against the ideal order (its own attempt counts) and no order."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1506_04651_b200 as P
c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = synth.CONFIGS[c]()
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
model = P.Model(dict(w.model, m=w.m))


def timed(x, order, cnt=None):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    st = P.rd_stats()
    torch.cuda.synchronize()
    ev[0].record(); P.rd_reaction_radau5_cells(x, model, 0.5 * w.dt, order=order, stats=st, cell_counters=cnt); ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]), st.as_dict()


def desc(c0):
    return (f"att/cell mean {c0.mean():.1f} p50 {np.percentile(c0,50):.0f} p99 {np.percentile(c0,99):.0f} max {c0.max()}")


for step in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    uu = g.values_view()
    n = uu.shape[1]
    u0 = uu.clone()
    cnt1 = torch.zeros((8, n), dtype=torch.int32, device="cuda")
    key = P.rd_reaction_cost(u0, model)
    oproxy = torch.argsort(key, descending=True, stable=True).to(torch.int32)
    for name, order in (("none", None), ("proxy", oproxy)):
        for rep in range(2):
            x = u0.clone(); ms, st = timed(x, order, cnt1)
        print(f"step {step} half 1 order={name:6s} n={n} ms={ms:.3f} attempts={st['n_attempts']} newton={st['n_newton']}")
    c1 = cnt1[0].clone()
    print("   half 1:", desc(c1.cpu().numpy()))
    oown = torch.argsort(c1, descending=True, stable=True).to(torch.int32)
    x = u0.clone(); ms, st = timed(x, oown)
    print(f"step {step} half 1 order=own    ms={ms:.3f}")
    uu.copy_(x)
    g.diffusion_rock4(w.eps_diff, w.dt)
    u1 = g.values_view().clone()
    cnt2 = torch.zeros((8, n), dtype=torch.int32, device="cuda")
    for name, order in (("none", None), ("half1", oown)):
        for rep in range(2):
            x = u1.clone(); ms, st = timed(x, order, cnt2)
        print(f"step {step} half 2 order={name:6s} ms={ms:.3f} attempts={st['n_attempts']} newton={st['n_newton']}")
    c2 = cnt2[0].clone()
    print("   half 2:", desc(c2.cpu().numpy()))
    key2 = P.rd_reaction_cost(u1, model)
    for name, order in (("own", torch.argsort(c2, descending=True, stable=True).to(torch.int32)),
                        ("proxy", torch.argsort(key2, descending=True, stable=True).to(torch.int32))):
        x = u1.clone(); ms, st = timed(x, order)
        print(f"step {step} half 2 order={name:6s} ms={ms:.3f}")
    cc1, cc2 = c1.cpu().numpy().astype(np.float64), c2.cpu().numpy().astype(np.float64)
    print(f"   corr(att1, att2) = {np.corrcoef(cc1, cc2)[0,1]:.3f}; cells with att2 > 2 att1: {(cc2 > 2*cc1).mean()*100:.1f} %")
    if os.environ.get("R5_DUMPK"):
        keys, _ = g.leaf_tensors()
        np.savez_compressed(f"{os.environ['R5_DUMPK']}_{step}.npz", keys=keys.cpu().numpy(), att1=cc1.astype(np.int16), att2=cc2.astype(np.int16),
                            key1=key.cpu().numpy().astype(np.int32), key2=key2.cpu().numpy().astype(np.int32))
    if os.environ.get("R5_DUMP"):
        rs = np.random.RandomState(step)
        idx = np.sort(rs.choice(n, size=min(n, 260000), replace=False))
        ti = torch.tensor(idx, device="cuda")
        np.savez(f"{os.environ['R5_DUMP']}_{step}.npz", idx=idx, u0=u0[:, ti].cpu().numpy(), u1=u1[:, ti].cpu().numpy(),
                 att1=cc1[idx].astype(np.int32), att2=cc2[idx].astype(np.int32), n=n)
    g.values_view().copy_(x)
    g.adapt()
