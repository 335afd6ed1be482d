"""Debug: one step of SymmetricShardedRBFGS vs RowShardedRBFGS on the GPU (development tool)."""
import numpy as np
import torch

import paper_1602_01768_b200 as si
from paper_1602_01768_b200 import generators as G
from paper_1602_01768_b200.dist import CudaPanelOps, RowShardedRBFGS, SymmetricShardedRBFGS

ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
ops = CudaPanelOps(ctx)
n, q = 600, 24
a = G.config1_dense(n, seed=4)
at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
sym = SymmetricShardedRBFGS(ops, n, q, lambda r0, r1: at[:, r0:r1].contiguous().reshape(-1), seed=3)
row = RowShardedRBFGS(ops, n, q, torch.from_numpy(a.reshape(-1, order="F").copy()).cuda(), seed=3)
x0s = sym.gather_x().cpu().numpy().reshape((n, n), order="F")
print("x0 identity", np.abs(x0s - np.eye(n)).max())
sym.step()
row.step()
torch.cuda.synchronize()
print("S", (sym.U[: n * q] - row.S).abs().max().item())
print("Y", (sym.Y - row.Y).abs().max().item())
print("W", (sym.U[n * q:] - row.U[n * q:]).abs().max().item())
print("P", (sym.P - row.P).abs().max().item(), row.P.abs().max().item())
print("M", (sym.M - row.M).abs().max().item())
xs = sym.gather_x().cpu().numpy().reshape((n, n), order="F")
xr = row.gather_x().cpu().numpy().reshape((n, n), order="F")
print("X", np.abs(xs - xr).max(), np.abs(xr).max())
d = np.abs(xs - xr)
print("err blocks", d[:300, :300].max(), d[:300, 300:].max(), d[300:, 300:].max())
for it in range(2, 6):
    sym.step(); row.step(); torch.cuda.synchronize()
    xs = sym.gather_x().cpu().numpy().reshape((n, n), order="F")
    xr = row.gather_x().cpu().numpy().reshape((n, n), order="F")
    d = np.abs(xs - xr)
    print(it, "W", (sym.U[n * q:] - row.U[n * q:]).abs().max().item(), "X", d.max(),
          d[:300, :300].max(), d[:300, 300:].max(), d[300:, 300:].max())
print("draws", sym.draw, row.draw, "redraws", sym.redraws, row.redraws)
sym2 = SymmetricShardedRBFGS(ops, n, q, lambda r0, r1: at[:, r0:r1].contiguous().reshape(-1), seed=3)
row2 = RowShardedRBFGS(ops, n, q, torch.from_numpy(a.reshape(-1, order="F").copy()).cuda(), seed=3)
for it in range(1, 4):
    sym2.step(); row2.step(); torch.cuda.synchronize()
    print(it, "P", (sym2.P - row2.P).abs().max().item(), "M", (sym2.M - row2.M).abs().max().item(),
          "V?", "draw", sym2.draw, row2.draw)
