"""Quick per-kernel timing of one RBFGS configuration (development tool)."""
import sys, time, json
import numpy as np
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = int(sys.argv[2]) if len(sys.argv) > 2 else 128
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
t0 = time.time()
if n >= 8192:
    # cheap SPD stand-in for timing only
    a = np.asfortranarray(np.eye(n) * 2.0)
else:
    a = G.config3_dense(n)
print("gen", time.time() - t0, flush=True)
prob = si.ProblemMatrix(a, si.Symmetry.spd)
sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=0)
sol.step(2)
ctx = prob.ctx
ctx.synchronize()
ctx.set_profiling(True)
ctx.reset_profile()
t0 = time.time()
sol.step(iters)
ctx.synchronize()
dt = time.time() - t0
prof = ctx.profile()
tot = sum(v[1] for v in prof.values())
print(f"n={n} q={q} iters={iters} wall {dt*1e3/iters:.3f} ms/iter; kernel sum {tot/iters:.3f} ms/iter")
F = 6.0 * n * n * q
for k, (l, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:20s} launches {l:6d}  {ms/iters:9.4f} ms/iter  {100*ms/tot:5.1f}%")
print("algorithmic TF/s (6n^2q per iter):", F / (tot / iters * 1e-3) / 1e12)
