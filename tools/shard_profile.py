"""Per-kernel-class device times of one RBFGS iteration, single-GPU solver vs the sharded
solver on a multi-GPU context of one GPU (NCCL) — diagnostic for the sharded path's
overhead.  Eager launches with per-launch CUDA events (no graphs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = 128
a = G.config3_dense(n, seed=0)
for name, ctx in (("single", si.Context(0)), ("sharded P=1", si.Context.multi([0])), ("loopback P=2", si.Context.loopback(0, 2))):
    prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
    s = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=0)
    s.step(3)
    ctx.set_profiling(True)
    ctx.reset_profile()
    s.step(5)
    prof = ctx.profile()
    ctx.set_profiling(False)
    tot = sum(v[1] for v in prof.values())
    print(f"== {name}: {tot / 5:.3f} ms of kernels per iteration (serialised, eager)")
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:22s} {v[0] / 5:5.1f} launches  {v[1] / 5:8.3f} ms")
    del s, prob
