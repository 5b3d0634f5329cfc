"""Scheduling-key study for the Radau5 thread kernel (BZ cells): times rd_reaction_radau5_cells with
explicit cell orders built from candidate keys (torch, on the device).  Usage: r5_keys.py cfg2|cfg4h1|cfg4h2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1506_04651_b200 as P
what = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
os.environ["RDMR_NO_PROXY_LPT"] = "1"  # only the explicit orders below
O = synth.OREGONATOR
spec = dict(kind="oregonator", **O)
model = P.Model(spec)
if what == "cfg2":
    w = synth.cfg2()
    u0 = torch.tensor(w.u.reshape(3, -1), device="cuda").contiguous()
    T = w.T if hasattr(w, "T") else 1e-2
else:
    w = synth.cfg4()
    u = torch.tensor(w.u.reshape(w.m, -1), device="cuda")
    g = P.Grid.build(w.dim, w.level_min, w.level_max, w.eps_mr, P.mr_rowmajor_to_morton(w.dim, w.level_max, u))
    g.strang_step(model, w.eps_diff, w.dt); g.adapt()   # a developed state
    T = 0.5 * w.dt
    if what == "cfg4h2":
        x = g.values_view().clone(); P.rd_reaction_radau5_cells(x, model, T); g.values_view().copy_(x)
        g.diffusion_rock4(w.eps_diff, w.dt)
    u0 = g.values_view().clone()
n = u0.shape[1]
print(what, "n =", n, "T =", T)


def timed(order, cnt=None):
    x = u0.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record(); P.rd_reaction_radau5_cells(x, model, T, order=order, cell_counters=cnt); ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1])


def order_of(*keys):
    """lexicographic descending by keys[0], then keys[1], ... (stable)"""
    o = torch.arange(n, device="cuda")
    for k in reversed(keys):
        o = o[torch.argsort(k[o], descending=True, stable=True)]
    return o.to(torch.int32)


a, b, c = u0
f = torch.stack([(-O["q"] * a - a * b + O["f_c"] * c) / O["mu"], (O["q"] * a - a * b + b * (1 - b)) / O["eps_b"], b - c])
r = f.abs() / (1e-8 + 1e-8 * u0.abs())
S = torch.log2(r.sum(0).clamp_min(1e-30))
L = torch.log2(r.clamp_min(1e-30))
lu = torch.log2(u0.abs().clamp_min(1e-30))
qz = lambda x, s: torch.floor(x / s)
cnt = torch.zeros((8, n), dtype=torch.int32, device="cuda")
timed(None, cnt); t_none = timed(None, cnt)
att, newt, lus = cnt[0].clone().double(), cnt[6].clone().double(), cnt[5].clone().double()
print(f"attempts/cell mean {att.mean():.1f} max {att.max():.0f}; newton/attempt {newt.sum()/att.sum():.2f}")
cands = {
    "none": None,
    "k16 proxy": order_of(qz(S, 1 / 64)),
    "k31 p.25,u1 .5,u0": order_of(qz(S, .25), qz(lu[1], .5), lu[0]),
    "own att": order_of(att),
    "own att,newt": order_of(att, newt),
    "own att,newt,lu": order_of(att, newt, lus),
    "p.5,u1 .5,u0": order_of(qz(S, .5), qz(lu[1], .5), lu[0]),
    "p1,u1 .5,u0": order_of(qz(S, 1.), qz(lu[1], .5), lu[0]),
    "p.25,u1 .25,u0": order_of(qz(S, .25), qz(lu[1], .25), lu[0]),
    "p.25,u1 1,u0": order_of(qz(S, .25), qz(lu[1], 1.), lu[0]),
    "p.25,u2 .5,u1 .5,u0": order_of(qz(S, .25), qz(lu[2], .5), qz(lu[1], .5), lu[0]),
    "p.25,u1 .5,u2 .5,u0": order_of(qz(S, .25), qz(lu[1], .5), qz(lu[2], .5), lu[0]),
    "p.25,u1 .5,u0 .5,u2": order_of(qz(S, .25), qz(lu[1], .5), qz(lu[0], .5), lu[2]),
    "p.25,u0 .5,u1": order_of(qz(S, .25), qz(lu[0], .5), lu[1]),
    "p.25,lb .5,la": order_of(qz(S, .25), qz(L[1], .5), L[0]),
    "p.5,u2 1,u1 .5,u0": order_of(qz(S, .5), qz(lu[2], 1.), qz(lu[1], .5), lu[0]),
    "state u2 .5,u1 .5,u0": order_of(qz(lu[2], .5), qz(lu[1], .5), lu[0]),
    "p2,u2 .5,u1 .5,u0": order_of(qz(S, 2.), qz(lu[2], .5), qz(lu[1], .5), lu[0]),
}
if len(sys.argv) > 2 and sys.argv[2] == "bits":  # integer keys as the kernel would build them, fewer radix passes
    cl = lambda x, lo, hi: torch.clamp(torch.floor(x), lo, hi)
    cands = {
        "none": None,
        "k31 (12,8@.5,11@1/16)": order_of(cl((S + 256) * 4, 0, 4095), cl((lu[1] + 64) * 2, 0, 255), cl((lu[0] + 64) * 16, 0, 2047)),
        "A31 (12,9@.25,10@1/8)": order_of(cl((S + 256) * 4, 0, 4095), cl((lu[1] + 64) * 4, 0, 511), cl((lu[0] + 64) * 8, 0, 1023)),
        "B24 (10,7@.5,7@.5)": order_of(cl((S + 100) * 4, 0, 1023), cl((lu[1] + 40) * 2, 0, 127), cl((lu[0] + 40) * 2, 0, 127)),
        "C24 (10,6@1,8@.25)": order_of(cl((S + 100) * 4, 0, 1023), cl((lu[1] + 40) * 1, 0, 63), cl((lu[0] + 40) * 4, 0, 255)),
        "D24 (10,8@.25,6@1)": order_of(cl((S + 100) * 4, 0, 1023), cl((lu[1] + 40) * 4, 0, 255), cl((lu[0] + 40) * 1, 0, 63)),
        "E16 (10,6@1)": order_of(cl((S + 100) * 4, 0, 1023), cl((lu[1] + 40) * 1, 0, 63)),
        "F16 (9@.5,7@.5)": order_of(cl((S + 100) * 2, 0, 511), cl((lu[1] + 40) * 2, 0, 127)),
        "G24 (9@.5,8@.25,7@.5)": order_of(cl((S + 100) * 2, 0, 511), cl((lu[1] + 40) * 4, 0, 255), cl((lu[0] + 40) * 2, 0, 127)),
    }
for name, o in cands.items():
    ts = [timed(o) for _ in range(2)]
    print(f"{name:28s} {min(ts):8.3f} ms", flush=True)
