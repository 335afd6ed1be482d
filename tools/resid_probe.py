"""Time the 2n^3 residual GEMM (||I - A X||_F) at config-3 size (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t = G.config3_dense_device(n, seed=0)
a = t.cpu().numpy().T
ctx = si.Context(0)
prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
x = np.asfortranarray(np.eye(n) * 0.5)
for r in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v = si.residual(prob, x)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"residual {v:.6e}  {1e3*dt:.1f} ms (incl. H2D of X {8*n*n/1e9:.2f} GB)", flush=True)
