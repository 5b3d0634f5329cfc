"""Does the previous Strang step's per-cell work (attempts, Newton iterations, LU pairs), carried through
the adaptation by leaf key, order this step's reaction half steps better than the stateless key?
Piecewise RDR steps on cfg 4 through the public calls; explicit orders; CUDA-event times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1506_04651_b200 as P
os.environ["RDMR_NO_PROXY_LPT"] = "1"
c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = synth.CONFIGS[c]()
D = w.dim
O = synth.OREGONATOR
model = P.Model(dict(w.model, m=w.m))
u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
T = 0.5 * w.dt


def timed(x0, order, cnt=None):
    x = x0.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record(); P.rd_reaction_radau5_cells(x, model, T, order=order, cell_counters=cnt); ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]), x


def order_of(n, *keys):
    o = torch.arange(n, device="cuda")
    for k in reversed(keys):
        o = o[torch.argsort(k[o], descending=True, stable=True)]
    return o.to(torch.int32)


def k31(u0):
    a, b, cc = u0
    f = torch.stack([(-O["q"] * a - a * b + O["f_c"] * cc) / O["mu"], (O["q"] * a - a * b + b * (1 - b)) / O["eps_b"], b - cc])
    S = torch.log2((f.abs() / (1e-8 + 1e-8 * u0.abs())).sum(0).clamp_min(1e-30))
    lu = torch.log2(u0.abs().clamp_min(1e-30))
    return torch.floor(S / .25), torch.floor(lu[1] / .5), lu[0]


def lookup(newk, oldk, oldv):
    """old leaf values at the new leaves: same key, else nearest ancestor, else first-descendant chain"""
    out = torch.full((len(newk), oldv.shape[1]), -1, dtype=oldv.dtype, device="cuda")
    todo = torch.ones(len(newk), dtype=torch.bool, device="cuda")
    lev, mor = newk >> 58, newk & ((1 << 58) - 1)
    for up in list(range(0, 8)) + [-d for d in range(1, 8)]:
        ll = lev - up
        m2 = (mor >> (D * up)) if up >= 0 else (mor << (D * -up))
        keys = (ll.clamp_min(0) << 58) | m2
        i = torch.searchsorted(oldk, keys).clamp_max(len(oldk) - 1)
        hit = todo & (oldk[i] == keys) & (ll >= 0)
        out[hit] = oldv[i[hit]]
        todo &= ~hit
    return out, todo


prev = None
for step in range(nsteps):
    keys, _ = g.leaf_tensors()
    uu = g.values_view(); n = uu.shape[1]
    u0 = uu.clone()
    res = {}
    cnt1 = torch.zeros((8, n), dtype=torch.int32, device="cuda")
    timed(u0, None, cnt1)
    sig1 = torch.stack([cnt1[0], cnt1[6], cnt1[5]], 1).double()
    orders1 = {"k31": order_of(n, *k31(u0)), "own": order_of(n, sig1[:, 0], sig1[:, 1], sig1[:, 2])}
    if prev is not None:
        h, miss = lookup(keys, prev[0], prev[1])
        p, s, t = k31(u0)
        orders1["hist"] = order_of(n, h[:, 0], h[:, 1], h[:, 2])
        orders1["hist att,k31"] = order_of(n, h[:, 0], s, t)
        orders1["hist att,newt,k31"] = order_of(n, h[:, 0], h[:, 1], s, t)
    for nm, o in orders1.items():
        res["h1 " + nm] = min(timed(u0, o)[0] for _ in range(2))
    _, x = timed(u0, orders1["k31"])
    uu.copy_(x)
    g.diffusion_rock4(w.eps_diff, w.dt)
    u1 = g.values_view().clone()
    cnt2 = torch.zeros((8, n), dtype=torch.int32, device="cuda")
    timed(u1, None, cnt2)
    sig2 = torch.stack([cnt2[0], cnt2[6], cnt2[5]], 1).double()
    orders2 = {"k31": order_of(n, *k31(u1)), "own": order_of(n, sig2[:, 0], sig2[:, 1], sig2[:, 2])}
    if prev is not None:
        h, miss = lookup(keys, prev[0], prev[2])
        p, s, t = k31(u1)
        orders2["hist"] = order_of(n, h[:, 0], h[:, 1], h[:, 2])
        orders2["hist att,k31"] = order_of(n, h[:, 0], s, t)
        orders2["hist att,newt,k31"] = order_of(n, h[:, 0], h[:, 1], s, t)
    for nm, o in orders2.items():
        res["h2 " + nm] = min(timed(u1, o)[0] for _ in range(2))
    _, x = timed(u1, orders2["k31"])
    g.values_view().copy_(x)
    print(f"step {step} n={n}: " + "  ".join(f"{k} {v:.3f}" for k, v in res.items()), flush=True)
    prev = (keys.clone(), sig1, sig2)
    g.adapt()
