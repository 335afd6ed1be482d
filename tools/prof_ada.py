"""AdaRBFGS iterations of config 2's shape (paper uniform sampler) for launch-list
profiling: `ncu --metrics gpu__time_duration.sum ... python tools/prof_ada.py` (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
q = int(sys.argv[2]) if len(sys.argv) > 2 else 64
it = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prob = si.ProblemMatrix(G.config2_dense(n, seed=0), si.Symmetry.spd)
sol = si.Solver(prob, si.Method.adarbfgs, si.SketchRule.adaptive_cols_uniform(q), seed=0)
sol.step(it)
prob.ctx.synchronize()
print("ok", prob.ctx.launch_count())
