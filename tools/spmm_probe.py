"""Time + check the CSR SpMM Y = A·P (si_spmm_csr_device) on the config-4 / config-5 matrices
(diagnostic).  SI_SPMM_ROWBLOCK=0 selects the warp-per-row kernel, SI_SPMM_NS the slabs per pass."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G
from paper_1602_01768_b200.dist import CudaPanelOps

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n, q = (98304, 512) if cfg == 5 else (65536, 256)
if len(sys.argv) > 2:
    n = int(sys.argv[2])
csr = G.config5_csr(n, half_bandwidth=64, seed=0) if cfg == 5 else G.config4_csr(n)
rowptr, colind, val = csr
ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
ops = CudaPanelOps(ctx)
dev = "cuda"
rp = torch.from_numpy(np.ascontiguousarray(rowptr, dtype=np.int64)).to(dev)
ci = torch.from_numpy(np.ascontiguousarray(colind, dtype=np.int32)).to(dev)
va = torch.from_numpy(np.ascontiguousarray(val, dtype=np.float64)).to(dev)
g = torch.Generator(device=dev).manual_seed(0)
P = torch.randn(q, n, dtype=torch.float64, device=dev, generator=g)  # column-major n×q
Y = torch.empty(q, n, dtype=torch.float64, device=dev)
ops.spmm(n, n, rp, ci, va, P, n, q, Y, n)
torch.cuda.synchronize()
# check a few columns against torch's sparse product
A = torch.sparse_csr_tensor(rp, ci.to(torch.int64), va, size=(n, n))
ref = (A @ P[:8].T.contiguous()).T
err = (Y[:8] - ref).abs().max().item() / ref.abs().max().item()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    ops.spmm(n, n, rp, ci, va, P, n, q, Y, n)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nnz = int(rowptr[-1])
alg = 12.0 * nnz + 8.0 * (n + 1) + 16.0 * n * q
print(f"config {cfg} n={n} q={q} nnz={nnz}: max rel err {err:.2e}; transpose + SpMM {ms:.3f} ms "
      f"({alg / ms / 1e6:.0f} GB/s algorithmic, {2.0 * nnz * q / ms / 1e9:.2f} TFLOP/s)", flush=True)
