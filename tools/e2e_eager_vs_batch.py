"""run_inverter at config 3: batched device loop vs SI_RUN_EAGER=1 (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G
n, q = 16384, 128
ctx = si.Context(0)
t = G.config3_dense_device(n, seed=0); a = t.cpu().numpy().T; del t
prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
def run(k, every):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian_device(q), tol=0.0, max_iters=k, seed=0,
                                          track=si.TrackOptions(residual_every_k=every), return_x=False))
    torch.cuda.synchronize(); return time.perf_counter() - t0, r
for mode in ("batch", "eager", "batch", "eager"):
    if mode == "eager": os.environ["SI_RUN_EAGER"] = "1"
    else: os.environ.pop("SI_RUN_EAGER", None)
    for k, every in ((1, 1), (2, 1000), (100, 100)):
        dt, r = run(k, every)
        print(f"{mode:6s} k={k:3d} every={every:4d}: {1e3*dt:8.1f} ms  seconds={r.state.seconds*1e3:8.1f} ms", flush=True)
