"""Row-sharded multi-GPU RBFGS, one process per GPU.

X (symmetric n×n) and dense A are split by rows: rank p owns rows
R_p = [r0_p, r1_p) as column-major panels X_p = X[R_p, :], A_p = A[R_p, :].
One iteration (SURVEY App. C1 rank-2q form):

    S        = Philox(seed, draw)            identical bytes on every rank (no traffic)
    Y_p      = A_p · S                       local DMMA GEMM        2·m·n·q
    Y        = all-gather(Y_p)               NCCL, n×q
    W_p      = X_p · Y                       local                  2·m·n·q
    P_p      = Y_pᵀ · [S_p  W_p]             local q×2q partial
    P        = all-reduce(P_p)               NCCL, 2q² doubles (G and YᵀW packed)
    M        = core(P)                       replicated q×q stage (Gram inverse + PD check)
    W        = all-gather(W_p)               NCCL, n×q
    V_p      = [S_p W_p] · M                 local
    X_p     += V_p · [S W]ᵀ                  local rank-2q update   4·m·n·q

Collectives go through torch.distributed (NCCL over NVLink on GPUs; gloo on
CPU for the host-logic tests); all arithmetic goes through `ops`, by default
the sm_100a C ABI (si_gemm_device, si_sketch_gaussian_device,
si_rbfgs_core_device, si_residual_rows_device).  The row-panel update does the
full m×n panel (4mnq) where the single-GPU path updates only upper tiles, so
the per-rank FLOPs are 8n²q/P against 6n²q on one GPU (documented in DESIGN.md).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib as L
from .api import GramRankDeficientError, ProblemMatrix, _check


def row_partition(n: int, world: int):
    """Rows per rank: contiguous, sizes differ by at most one."""
    base, extra = divmod(n, world)
    starts, r = [], 0
    for p in range(world):
        starts.append(r)
        r += base + (1 if p < extra else 0)
    starts.append(n)
    return starts


class CudaPanelOps:
    """Panel operations on CUDA tensors through libstochinv_b200 (no fallback)."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.lib = L.load()

    @staticmethod
    def _p(t: torch.Tensor):
        return C.c_void_p(t.data_ptr())

    def gemm(self, M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, Cm, ldc, alpha=1.0, beta=0.0):
        _check(self.lib.si_gemm_device(self.ctx.handle, M, N, K, self._p(A), lda, int(a_kmajor), self._p(B), ldb,
                                       int(b_kmajor), self._p(Cm), ldc, float(alpha), float(beta)))

    def sketch(self, S, n, q, lds, seed, draw):
        _check(self.lib.si_sketch_gaussian_device(self.ctx.handle, self._p(S), n, q, lds, C.c_uint64(seed),
                                                  C.c_uint64(draw)))

    def core(self, P, ldp, q, M, scratch):
        _check(self.lib.si_rbfgs_core_device(self.ctx.handle, self._p(P), ldp, q, self._p(M), self._p(scratch)))

    def residual_rows_sq(self, prob: ProblemMatrix, m, r0, X, ldx) -> float:
        out = C.c_double()
        _check(self.lib.si_residual_rows_device(self.ctx.handle, prob.handle, m, r0, self._p(X), ldx, C.byref(out)))
        return out.value


@dataclass
class ShardLayout:
    n: int
    q: int
    rank: int
    world: int

    def __post_init__(self):
        self.starts = row_partition(self.n, self.world)
        self.r0 = self.starts[self.rank]
        self.r1 = self.starts[self.rank + 1]
        self.m = self.r1 - self.r0
        self.m_max = max(self.starts[p + 1] - self.starts[p] for p in range(self.world))


class RowShardedRBFGS:
    """RBFGS with X row-sharded over the ranks of the default process group.

    a_rows: A[R_p, :] as a column-major m×n panel held in a flat float64 tensor
    (on the ops' device).  `prob` (optional) is a ProblemMatrix with the full
    dense A on this rank's GPU, used only by the residual.
    """

    def __init__(self, ops, n: int, q: int, a_rows: torch.Tensor, *, seed: int = 0, device=None,
                 prob: ProblemMatrix | None = None, max_redraws: int = 100):
        self.ops = ops
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.lay = ShardLayout(n, q, self.rank, self.world)
        self.seed = seed
        self.draw = 0
        self.prob = prob
        self.max_redraws = max_redraws
        self.redraws = 0
        dev = device if device is not None else a_rows.device
        m, mm = self.lay.m, self.lay.m_max
        f = dict(dtype=torch.float64, device=dev)
        self.A = a_rows
        self.X = torch.zeros(m * n, **f)
        self.S = torch.empty(n * q, **f)
        self.Y = torch.empty(n * q, **f)
        self.Yp = torch.empty(m * q, **f)
        self.Up = torch.empty(m * 2 * q, **f)  # [S_p W_p]
        self.U = torch.empty(n * 2 * q, **f)   # [S W]
        self.P = torch.empty(q * 2 * q, **f)
        self.M = torch.empty(4 * q * q, **f)
        self.Vp = torch.empty(m * 2 * q, **f)
        self.scratch = torch.empty(6 * q * q + 2 * q + 16, **f)
        self.gather_buf = torch.empty(self.world * mm * q, **f)
        self.send_buf = torch.zeros(mm * q, **f)
        self.set_identity()

    # ------------------------------------------------------------- layout --
    def set_identity(self):
        lay = self.lay
        Xv = self.X.view(lay.n, lay.m)  # column-major m×n  ==  row-major (n, m)
        Xv.zero_()
        idx = torch.arange(lay.m, device=self.X.device)
        Xv[lay.r0 + idx, idx] = 1.0

    def set_rows(self, x_rows: torch.Tensor):
        """x_rows: column-major m×n panel (flat)."""
        self.X.copy_(x_rows)

    def _all_gather_rows(self, panel: torch.Tensor, out: torch.Tensor, ncols: int):
        """panel: this rank's m×ncols column-major panel; out: n×ncols column-major."""
        lay = self.lay
        mm = lay.m_max
        send = self.send_buf[: mm * ncols].view(ncols, mm)
        send[:, : lay.m].copy_(panel.view(ncols, lay.m))
        if self.world == 1:
            out.view(ncols, lay.n).copy_(send[:, : lay.n])
            return
        gbuf = self.gather_buf[: self.world * mm * ncols]
        dist.all_gather_into_tensor(gbuf, send.reshape(-1))
        g = gbuf.view(self.world, ncols, mm)
        ov = out.view(ncols, lay.n)
        for p in range(self.world):
            a, b = lay.starts[p], lay.starts[p + 1]
            ov[:, a:b].copy_(g[p, :, : b - a])

    # --------------------------------------------------------------- step --
    def step(self):
        """One iteration; a rejected Gram (not PD on every rank alike) is redrawn."""
        lay, ops = self.lay, self.ops
        n, q, m = lay.n, lay.q, lay.m
        for attempt in range(self.max_redraws + 1):
            draw = self.draw
            self.draw += 1
            ops.sketch(self.S, n, q, n, self.seed, draw)
            ops.gemm(m, q, n, self.A, m, False, self.S, n, True, self.Yp, m)           # Y_p = A_p·S
            self._all_gather_rows(self.Yp, self.Y, q)                                   # Y
            Sv = self.S.view(q, n)
            Upv = self.Up.view(2 * q, m)
            Upv[:q].copy_(Sv[:, lay.r0:lay.r1])                                         # S_p
            Wp = self.Up[m * q:]
            ops.gemm(m, q, n, self.X, m, False, self.Y, n, True, Wp, m)                 # W_p = X_p·Y
            ops.gemm(q, 2 * q, m, self.Yp, m, True, self.Up, m, True, self.P, q)        # P_p = Y_pᵀ·[S_p W_p]
            if self.world > 1:
                dist.all_reduce(self.P)                                                 # packed [G | YᵀW]
            try:
                ops.core(self.P, q, q, self.M, self.scratch)                            # M (replicated)
            except GramRankDeficientError:
                self.redraws += 1  # same P on every rank -> every rank redraws together
                continue
            Uv = self.U.view(2 * q, n)
            Uv[:q].copy_(Sv)
            self._all_gather_rows(Wp, self.U[n * q:], q)                                # W
            ops.gemm(m, 2 * q, 2 * q, self.Up, m, False, self.M, 2 * q, True, self.Vp, m)  # V_p = U_p·M
            ops.gemm(m, n, 2 * q, self.Vp, m, False, self.U, n, False, self.X, m, 1.0, 1.0)  # X_p += V_p·Uᵀ
            return
        raise GramRankDeficientError("sketch rejection limit exceeded")

    def residual(self) -> float:
        """‖I − A X‖_F from the row panels (= ‖I − X A‖_F, A and X symmetric)."""
        lay = self.lay
        part = self.ops.residual_rows_sq(self.prob, lay.m, lay.r0, self.X, lay.m)
        t = torch.tensor([part], dtype=torch.float64, device=self.X.device)
        if self.world > 1:
            dist.all_reduce(t)
        return float(t.item()) ** 0.5

    def gather_x(self) -> torch.Tensor:
        """Full X (n×n column-major, flat) on every rank (tests / export)."""
        out = torch.empty(self.lay.n * self.lay.n, dtype=torch.float64, device=self.X.device)
        self._gather_full(out)
        return out

    def _gather_full(self, out):
        lay = self.lay
        mm = lay.m_max
        send = torch.zeros(mm * lay.n, dtype=torch.float64, device=self.X.device).view(lay.n, mm)
        send[:, : lay.m].copy_(self.X.view(lay.n, lay.m))
        if self.world == 1:
            out.view(lay.n, lay.n).copy_(send[:, : lay.n])
            return
        g = torch.empty(self.world * mm * lay.n, dtype=torch.float64, device=self.X.device)
        dist.all_gather_into_tensor(g, send.reshape(-1))
        gv = g.view(self.world, lay.n, mm)
        ov = out.view(lay.n, lay.n)
        for p in range(self.world):
            a, b = lay.starts[p], lay.starts[p + 1]
            ov[:, a:b].copy_(gv[p, :, : b - a])
