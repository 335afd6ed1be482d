"""Step the AdaRBFGS solver at config 2 (diagnostic, for ncu captures)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n, q = 4096, 64
ctx = si.Context(0)
prob = si.ProblemMatrix(G.config2_dense(n, seed=0), si.Symmetry.spd, context=ctx)
sol = si.Solver(prob, si.Method.adarbfgs, si.SketchRule.adaptive_cols_uniform(q), seed=0)
sol.step(3)
torch.cuda.synchronize()
t0 = time.perf_counter(); sol.step(steps); torch.cuda.synchronize()
print(f"config 2: {1e3*(time.perf_counter()-t0)/steps:.4f} ms/iter", flush=True)
