"""First steps after bench.py's restart(): per-phase times (R, D, A) of each step, to find one-off costs
of a fresh grid.  usage: python tools/first_step.py [cfg] [warmup] [steps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1506_04651_b200 as P

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 4
torch.cuda.set_device(0)
W = bench.WORKLOADS[cfg](P, torch, 0)
for _ in range(nw):
    W.step()
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.time()
    W.restart()
    torch.cuda.synchronize()
    print(f"restart {1e3 * (time.time() - t0):.1f} ms wall", flush=True)
    for k in range(ns):
        W.phase_ms = {"R": 0.0, "D": 0.0, "A": 0.0}
        t0 = time.time()
        ms = W.step(timed=True)
        print(f"  step {k}: device {ms:.2f} ms, wall {1e3 * (time.time() - t0):.2f} ms, R {W.phase_ms['R']:.2f} D {W.phase_ms['D']:.2f} A {W.phase_ms['A']:.2f}", flush=True)
