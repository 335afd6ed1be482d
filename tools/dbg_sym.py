"""Debug: the symmetric sharded driver's GPU ops against numpy (development tool)."""
import numpy as np
import torch

import paper_1602_01768_b200 as si
from paper_1602_01768_b200.dist import CudaPanelOps

ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
ops = CudaPanelOps(ctx)
rng = np.random.default_rng(0)
n, q, m, r0 = 600, 24, 300, 0
r1 = r0 + m


def dev(x):
    return torch.from_numpy(np.asarray(x).reshape(-1, order="F").copy()).cuda()


def host(t, rows, cols, ld=None):
    a = t.cpu().numpy()
    ld = ld or rows
    return np.lib.stride_tricks.as_strided(a, shape=(rows, cols), strides=(8, 8 * ld)).copy()


Xc = rng.standard_normal((m, n - r0))
Y = rng.standard_normal((n, q))
W0 = rng.standard_normal((n, q))
# 1) W[r0:] += Xc·Y[r0:]
W = dev(W0); Yd = dev(Y); Xd = dev(Xc)
ops.gemm(m, q, n - r0, Xd, m, False, Yd[r0:], n, True, W[r0:], n, 1.0, 1.0)
torch.cuda.synchronize()
ref = W0.copy(); ref[r0:r1] += Xc @ Y[r0:]
print("gemm1", np.abs(host(W, n, q) - ref).max())
# 2) W[r1:] += Xc[:, m:]ᵀ·Y[r0:r1]
W = dev(W0)
ops.gemm(n - r1, q, m, Xd[m * m:], m, True, Yd[r0:], n, True, W[r1:], n, 1.0, 1.0)
torch.cuda.synchronize()
ref = W0.copy(); ref[r1:] += Xc[:, m:].T @ Y[r0:r1]
print("gemm2", np.abs(host(W, n, q) - ref).max())
# 3) symupd X_c[:, :m] += V·U[r0:r1]ᵀ
U = rng.standard_normal((n, 2 * q)); V = rng.standard_normal((m, 2 * q))
S = rng.standard_normal((m, m)); S = S + S.T
Xs = np.zeros((m, n - r0)); Xs[:, :m] = S
Xd = dev(Xs); Ud = dev(U); Vd = dev(V)
ops.symupd(m, 2 * q, Vd, m, Ud[r0:], n, Xd, m)
torch.cuda.synchronize()
full = S + V @ U[r0:r1].T
refs = np.triu(full) + np.triu(full, 1).T
print("symupd", np.abs(host(Xd, m, n - r0)[:, :m] - refs).max())
# 4) X_c[:, m:] += V·U[r1:]ᵀ
Xs2 = rng.standard_normal((m, n - r0)); Xd = dev(Xs2)
ops.gemm(m, n - r1, 2 * q, Vd, m, False, Ud[r1:], n, False, Xd[m * m:], m, 1.0, 1.0)
torch.cuda.synchronize()
ref = Xs2.copy(); ref[:, m:] += V @ U[r1:].T
print("gemm4", np.abs(host(Xd, m, n - r0) - ref).max())
# 5) P += Y[r0:]ᵀ·U[r0:]
P0 = rng.standard_normal((q, 2 * q)); Pd = dev(P0)
ops.gemm(q, 2 * q, m, Yd[r0:], n, True, Ud[r0:], n, True, Pd, q, 1.0, 1.0)
torch.cuda.synchronize()
print("gemm5", np.abs(host(Pd, q, 2 * q) - (P0 + Y[r0:r1].T @ U[r0:r1])).max())
# 6) V = U[r0:]·M
M = rng.standard_normal((2 * q, 2 * q)); Md = dev(M); Vo = torch.empty(m * 2 * q, dtype=torch.float64, device="cuda")
ops.gemm(m, 2 * q, 2 * q, Ud[r0:], n, False, Md, 2 * q, True, Vo, m)
torch.cuda.synchronize()
print("gemm6", np.abs(host(Vo, m, 2 * q) - U[r0:r1] @ M).max())
# 7) Y[r0:] = A_c·S
A = rng.standard_normal((m, n)); Sm = rng.standard_normal((n, q)); Ad = dev(A); Sd = dev(Sm)
Yo = dev(np.zeros((n, q)))
ops.gemm(m, q, n, Ad, m, False, Sd, n, True, Yo[r0:], n)
torch.cuda.synchronize()
print("gemm7", np.abs(host(Yo, n, q)[r0:r1] - A @ Sm).max())
