"""Phase timing of the config-3 end-to-end run (diagnostic; not part of the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G

n, q = 16384, 128
ctx = si.Context(0)
a_dev = G.config3_dense_device(n, seed=0)
a_host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
a_host.copy_(a_dev)
a_np = a_host.numpy().T
del a_dev
torch.cuda.synchronize()

def t(label, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label:40s} {1e3*(time.perf_counter()-t0):9.1f} ms", flush=True)
    return r

prob = t("ProblemMatrix (H2D + sym + validate)", lambda: si.ProblemMatrix(a_np, si.Symmetry.spd, context=ctx))
x_pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
x_out = x_pinned.numpy().T
def run(k, every, ret=True, out=None):
    return si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian_device(q), tol=0.0, max_iters=k, seed=0,
                                             track=si.TrackOptions(residual_every_k=every), return_x=ret), out=out)
t("run 1 iter (k=1 checkpoint), no X", lambda: run(1, 1, False))
t("run 1 iter again", lambda: run(1, 1, False))
t("run 2 iters (k=1,2 checkpoints), no X", lambda: run(2, 1, False))
t("run 10 iters, every 1000 (k=1,10), no X", lambda: run(10, 1000, False))
t("run 100 iters every 100, no X", lambda: run(100, 100, False))
r = t("run 100 iters every 100, X out", lambda: run(100, 100, True, x_out))
print([(h.k, h.residual) for h in r.state.history])
xx = torch.from_numpy(np.ascontiguousarray(x_out.T))
t("residual (2n^3)", lambda: si.residual(prob, x_out))
