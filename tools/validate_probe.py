"""validate_spd on the engine's blocked Schur-complement test (diagnostic): SPD and
non-SPD inputs of several sizes, single-GPU and loopback contexts; times n = 16384."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1602_01768_b200 as si
from oracle import oracle as O

for n in (5, 120, 130, 300, 1000):
    b = O.RngStream(n).gaussian_matrix(n, n)
    a = b @ b.T / n + 0.5 * np.eye(n)
    for label, m in (("spd", a), ("neg00", a - np.diag([2.0] + [0.0] * (n - 1))),
                     ("neglast", a - np.diag([0.0] * (n - 1) + [50.0])), ("zero", np.zeros((n, n)))):
        for ctxname, ctx in (("single", si.Context(0)), ("loopback2", si.Context.loopback(0, 2))):
            p = si.ProblemMatrix(m, si.Symmetry.spd, context=ctx)
            try:
                p.validate_spd()
                ok = "pass"
            except Exception as e:
                ok = f"raise {type(e).__name__}: {e}"
            print(f"n={n:5d} {label:8s} {ctxname:10s} {ok}", flush=True)
if len(sys.argv) > 1:
    n = int(sys.argv[1])
    b = O.RngStream(1).gaussian_matrix(n, 64)
    a = np.asfortranarray(b @ b.T / 64 + np.eye(n))
    p = si.ProblemMatrix(a, si.Symmetry.spd)
    t0 = time.perf_counter(); p.validate_spd(); t1 = time.perf_counter()
    print(f"validate_spd n={n}: {1e3 * (t1 - t0):.1f} ms (first call, includes workspace)")
    p2 = si.ProblemMatrix(a, si.Symmetry.spd)
    t0 = time.perf_counter(); p2.validate_spd(); t1 = time.perf_counter()
    print(f"validate_spd n={n}: {1e3 * (t1 - t0):.1f} ms")
