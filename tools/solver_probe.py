"""Step the device-sketch RBFGS solver on a BASELINE config (diagnostic, for ncu launch lists)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if cfgn == 1:
    n, q = 1024, 32
    a = G.config1_dense(n, seed=0)
else:
    n, q = 16384, 128
    t = G.config3_dense_device(n, seed=0)
    a = t.cpu().numpy().T
ctx = si.Context(0)
prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=0)
sol.step(5)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    sol.step(steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"config {cfgn}: {1e3*dt/steps:.4f} ms/iter (wall, {steps} graph-replayed iterations)", flush=True)
