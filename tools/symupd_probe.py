"""Time K-SYMUPD (si_symupd_device) on config-3 shapes: separate vs windowed operands (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200.dist import CudaPanelOps

n, q = 16384, 128
ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
ops = CudaPanelOps(ctx)
X = torch.randn(n, n, dtype=torch.float64, device="cuda"); X = X + X.T
V = torch.randn(2 * q, n, dtype=torch.float64, device="cuda") * 1e-3
U = torch.randn(2 * q, n, dtype=torch.float64, device="cuda") * 1e-3
B5 = torch.randn(4 * q, n, dtype=torch.float64, device="cuda") * 1e-3
def run(label, Vt, Ut, reps=10):
    ops.symupd(n, 2 * q, Vt, n, Ut, n, X, n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.symupd(n, 2 * q, Vt, n, Ut, n, X, n)
    e1.record(); torch.cuda.synchronize()
    print(f"{label:40s} {e0.elapsed_time(e1)/reps:.3f} ms  (neg={os.environ.get('SI_SYMUPD_NEG')})", flush=True)
run("separate V, U", V, U)
run("windows [Z R], [W Z] of one buffer", B5[2 * q:], B5[q:3 * q])
run("separate V, U again", V, U)
