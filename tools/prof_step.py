"""Two RBFGS iterations of one config (for ncu: skip the first iteration's launches)."""
import sys
import numpy as np
import paper_1602_01768_b200 as si

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = int(sys.argv[2]) if len(sys.argv) > 2 else 128
a = np.asfortranarray(np.eye(n) * 2.0)
a[0, 1] = a[1, 0] = 0.5
prob = si.ProblemMatrix(a, si.Symmetry.spd)
sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=0)
sol.step(1)
sol.step(1)
prob.ctx.synchronize()
print("ok", prob.ctx.launch_count())
