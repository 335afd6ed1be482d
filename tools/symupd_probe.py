"""Time + check K-SYMUPD (si_symupd_device) on config-3 shapes (diagnostic).
SI_SYMUPD_TILE selects the variant (default / pp / 128x64 ...)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200.dist import CudaPanelOps

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = int(sys.argv[2]) if len(sys.argv) > 2 else 128
ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
ops = CudaPanelOps(ctx)
g = torch.Generator(device="cuda").manual_seed(0)
X0 = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g); X0 = X0 + X0.T
V = torch.randn(2 * q, n, dtype=torch.float64, device="cuda", generator=g) * 1e-3  # column-major n×2q
U = torch.randn(2 * q, n, dtype=torch.float64, device="cuda", generator=g) * 1e-3
# correctness: one update against torch (upper triangle of X0 + V·Uᵀ, mirrored)
X = X0.clone()  # X[i][j] row-major of a symmetric matrix == column-major
ops.symupd(n, 2 * q, V, n, U, n, X, n)
torch.cuda.synchronize()
Vc, Uc = V.T, U.T  # n×2q
ref = X0.T + Vc @ Uc.T  # column-major X(r, c) = X.T[r, c]
up = torch.triu(ref)
ref = up + torch.triu(up, 1).T
err = (X.T - ref).abs().max().item() / ref.abs().max().item()
sym = (X - X.T).abs().max().item()
print(f"variant={os.environ.get('SI_SYMUPD_TILE', 'default')} n={n} q={q} max rel err {err:.3e} asym {sym:.1e}", flush=True)
reps = 10
ops.symupd(n, 2 * q, V, n, U, n, X, n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ops.symupd(n, 2 * q, V, n, U, n, X, n)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"  {ms:.3f} ms  ({2.0 * n * n * 2 * q / 2 / (ms * 1e-3) / 1e12:.2f} TFLOP/s on the upper triangle)", flush=True)
