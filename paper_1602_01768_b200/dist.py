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
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

import numpy as np

from . import _lib as L
from .api import GramRankDeficientError, NumericalError, ProblemMatrix, RngStream, _check, contiguous_partition


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
    """Panel operations on CUDA tensors through libstochinv_b200 (no fallback).

    The drivers below interleave these launches with torch ops (copies, fills, NCCL
    collectives, event records) and rely on stream order between the two, so the context
    must launch on torch's current stream — create it as
    ``Context(device, stream=torch.cuda.current_stream().cuda_stream)`` — and the current
    torch stream must not change while a driver is in use.  A context on any other stream
    (e.g. ``Context(device)``'s private non-blocking stream) would race the torch ops, and
    is rejected here."""

    def __init__(self, ctx):
        cur = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
        if cur is not None and getattr(ctx, "stream", None) != cur:
            raise ValueError("CudaPanelOps: the context must launch on torch's current stream "
                             "(Context(device, stream=torch.cuda.current_stream().cuda_stream))")
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

    def core_async(self, P, ldp, q, M, scratch, status):
        """core() without the host read: status (device int32) = 0 when G is PD, M = 0 otherwise."""
        _check(self.lib.si_rbfgs_core_device_async(self.ctx.handle, self._p(P), ldp, q, self._p(M),
                                                   self._p(scratch), self._p(status)))

    def gather_columns(self, Lp, rows, ldl, idx, q, out):
        _check(self.lib.si_gather_columns_device(self.ctx.handle, self._p(Lp), rows, ldl, self._p(idx), q,
                                                 self._p(out)))

    def ada_core(self, G, q, Z, n, idx, St, T, R, B, scratch):
        _check(self.lib.si_ada_core_device(self.ctx.handle, self._p(G), q, self._p(Z), n,
                                           self._p(idx) if idx is not None else None,
                                           self._p(St) if St is not None else None,
                                           self._p(T) if T is not None else None, self._p(R), self._p(B),
                                           self._p(scratch)))

    def pdiag_update(self, B, q, n, T, idx, d):
        _check(self.lib.si_pdiag_update_device(self.ctx.handle, self._p(B), q, n,
                                               self._p(T) if T is not None else None,
                                               self._p(idx) if idx is not None else None, self._p(d)))

    def spmm(self, m, n, rowptr, colind, val, P, ldp, k, Y, ldy):
        _check(self.lib.si_spmm_csr_device(self.ctx.handle, m, n, self._p(rowptr), self._p(colind), self._p(val),
                                           self._p(P), ldp, k, self._p(Y), ldy))

    def symupd(self, m, k, V, ldv, U, ldu, X, ldx):
        _check(self.lib.si_symupd_device(self.ctx.handle, m, k, self._p(V), ldv, self._p(U), ldu, self._p(X), ldx))

    def residual_rows_sq(self, prob: ProblemMatrix, m, r0, X, ldx) -> float:
        out = C.c_double()
        _check(self.lib.si_residual_rows_device(self.ctx.handle, prob.handle, m, r0, self._p(X), ldx, C.byref(out)))
        return out.value


@dataclass
class CsrRows:
    """Rows [r0, r1) of a sparse A as a device CSR panel: rowptr relative to the
    panel (int64, m+1), global column indices (int32), values (float64)."""
    rowptr: torch.Tensor
    colind: torch.Tensor
    val: torch.Tensor
    r0: int
    m: int

    @staticmethod
    def from_host(rowptr, colind, val, r0: int, r1: int, device) -> "CsrRows":
        b, e = int(rowptr[r0]), int(rowptr[r1])
        rp = torch.from_numpy(np.asarray(rowptr[r0:r1 + 1], dtype=np.int64) - b).to(device)
        ci = torch.from_numpy(np.ascontiguousarray(colind[b:e], dtype=np.int32)).to(device)
        va = torch.from_numpy(np.ascontiguousarray(val[b:e], dtype=np.float64)).to(device)
        return CsrRows(rp, ci, va, r0, r1 - r0)

    def diagonal(self) -> torch.Tensor:
        """A[r0 + i, r0 + i] for the panel's rows (length m)."""
        counts = (self.rowptr[1:] - self.rowptr[:-1]).to(torch.int64)
        rows = torch.repeat_interleave(torch.arange(self.m, device=self.val.device), counts)
        d = torch.zeros(self.m, dtype=torch.float64, device=self.val.device)
        hit = self.colind.to(torch.int64) == rows + self.r0
        d.index_add_(0, rows[hit], self.val[hit])
        return d


def apply_rows(ops, A, n: int, P, ldp: int, k: int, out, ldo: int):
    """out (m×k, ld ldo) = A_rows·P for a dense column-major m×n panel (flat tensor, ld m)
    or a CsrRows panel; P is n×k (ld ldp)."""
    if isinstance(A, CsrRows):
        ops.spmm(A.m, n, A.rowptr, A.colind, A.val, P, ldp, k, out, ldo)
    else:
        m = A.numel() // n
        ops.gemm(m, k, n, A, m, False, P, ldp, True, out, ldo)


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


class _RowPanels:
    """Collectives on row panels shared by the sharded drivers (self.lay, self.world,
    self.send_buf / self.gather_buf sized for m_max × q)."""

    def _all_gather_rows(self, panel: torch.Tensor, out: torch.Tensor, ncols: int):
        """panel: this rank's m×ncols column-major panel; out: n×ncols column-major."""
        lay = self.lay
        mm = lay.m_max
        if self.world == 1:
            out[: lay.n * ncols].copy_(panel[: lay.n * ncols])
            return
        send = self.send_buf[: mm * ncols].view(ncols, mm)
        send[:, : lay.m].copy_(panel.view(ncols, lay.m))
        gbuf = self.gather_buf[: self.world * mm * ncols]
        dist.all_gather_into_tensor(gbuf, send.reshape(-1))
        # (P, ncols, mm) -> out's rows: one transposing copy when the panels are equal, else
        # the valid columns picked by one index_select (instead of P strided copies)
        cols = gbuf.view(self.world, ncols, mm).permute(1, 0, 2).reshape(ncols, self.world * mm)
        ov = out.view(ncols, lay.n)
        if self.world * mm == lay.n:
            ov.copy_(cols)
            return
        if getattr(self, "_row_src", None) is None or self._row_src.device != out.device:
            src = [p * mm + i for p in range(self.world) for i in range(lay.starts[p + 1] - lay.starts[p])]
            self._row_src = torch.tensor(src, dtype=torch.int64, device=out.device)
        ov.copy_(cols.index_select(1, self._row_src))

    def _gather_panel(self, panel, out):
        """All-gather an m×n row panel (column-major, flat) into the full n×n matrix."""
        lay = self.lay
        mm = lay.m_max
        send = torch.zeros(mm * lay.n, dtype=torch.float64, device=panel.device).view(lay.n, mm)
        send[:, : lay.m].copy_(panel.view(lay.n, lay.m))
        if self.world == 1:
            out.view(lay.n, lay.n).copy_(send[:, : lay.n])
            return
        g = torch.empty(self.world * mm * lay.n, dtype=torch.float64, device=panel.device)
        dist.all_gather_into_tensor(g, send.reshape(-1))
        gv = g.view(self.world, lay.n, mm)
        ov = out.view(lay.n, lay.n)
        for p in range(self.world):
            a, b = lay.starts[p], lay.starts[p + 1]
            ov[:, a:b].copy_(gv[p, :, : b - a])


class RowShardedRBFGS(_RowPanels):
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
        dev = device if device is not None else (a_rows.val.device if isinstance(a_rows, CsrRows) else a_rows.device)
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

    # --------------------------------------------------------------- step --
    def step(self):
        """One iteration; a rejected Gram (not PD on every rank alike) is redrawn."""
        lay, ops = self.lay, self.ops
        n, q, m = lay.n, lay.q, lay.m
        for attempt in range(self.max_redraws + 1):
            draw = self.draw
            self.draw += 1
            ops.sketch(self.S, n, q, n, self.seed, draw)
            apply_rows(ops, self.A, n, self.S, n, q, self.Yp, m)                         # Y_p = A_p·S
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
        self._gather_panel(self.X, out)


class RowShardedAdaRBFGS(_RowPanels):
    """AdaRBFGS with the factor L row-sharded: rank p owns the
    column-major m×n panel L_p = L[R_p, :] and A_p = A[R_p, :].  One iteration
    (adarbfgs.cpp:12-21 over panels):

        C / S̃    host draw (RngStream, identical on every rank) or Philox S̃
        S_p      = L_p[:, C]  or  L_p·S̃                    local
        S        = all-gather(S_p)                          n×q
        (AS)_p   = A_p·S                                    local  2·m·n·q
        [G | Z]  = all-reduce([S_pᵀ(AS)_p | (AS)_pᵀL_p])     q×q + q×n, one packed call
        R, B     = G^{-1/2},  T − R·Z                        replicated q×n stage
        L_p     += (S_p·R)·B                                 local  2·m·n·q
        d       += 2⟨T_j, B_j⟩ − ‖B_j‖²                      replicated Eq. 8.2 diagonal (App. C3)

    rule: "cols" (reference contiguous blocks + Eq. 8.2, adarbfgs.cpp:23-36),
    "uniform" (paper sampler, uniform q-subsets) or "gauss" (Philox S̃).  The host
    RNG consumption matches run_adarbfgs (one categorical / subset per attempt),
    so the coordinate paths draw the same indices as the single-GPU driver.
    """

    def __init__(self, ops, n: int, q: int, a_rows: torch.Tensor, *, rule: str = "cols", seed: int = 0,
                 prob: ProblemMatrix | None = None, max_redraws: int = 100, l0_rows: torch.Tensor | None = None):
        if rule not in ("cols", "uniform", "gauss"):
            raise ValueError("rule must be 'cols', 'uniform' or 'gauss'")
        self.ops, self.rule, self.seed, self.prob, self.max_redraws = ops, rule, seed, prob, max_redraws
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.lay = ShardLayout(n, q, self.rank, self.world)
        self.rng = RngStream(seed)
        self.draw = 0
        self.redraws = 0
        self.k = 0
        dev = a_rows.val.device if isinstance(a_rows, CsrRows) else a_rows.device
        m = self.lay.m
        f = dict(dtype=torch.float64, device=dev)
        self.A = a_rows
        self.L = torch.empty(m * n, **f)
        self.Sp = torch.empty(m * q, **f)
        self.S = torch.empty(n * q, **f)
        self.ASp = torch.empty(m * q, **f)
        self.SRp = torch.empty(m * q, **f)
        self.GZ = torch.empty(q * q + q * n, **f)
        self.R = torch.empty(q * q, **f)
        self.B = torch.empty(q * n, **f)
        self.scratch = torch.empty(8 * q * q + 8 * q + 32, **f)
        self.idx = torch.zeros(q, dtype=torch.int64, device=dev)
        # pinned staging for the host-drawn indices (a pageable H2D copy would synchronize the
        # stream at the start of every step); 4 slots, each reused only after the ada_core
        # status reads of the attempts in between
        self._idx_host = torch.zeros((4, q), dtype=torch.int64, pin_memory=self.idx.is_cuda)
        self._idx_slot = 0
        self.St = torch.empty(n * q, **f) if rule == "gauss" else None
        self.T = torch.empty(q * n, **f) if rule == "gauss" else None
        self.gather_buf = torch.empty(self.world * self.lay.m_max * q, **f)
        self.send_buf = torch.zeros(self.lay.m_max * q, **f)
        self.blocks = contiguous_partition(n, q) if rule == "cols" else None
        self.d = torch.empty(n, **f) if rule == "cols" else None
        if l0_rows is None:
            Lv = self.L.view(n, m)
            Lv.zero_()
            i = torch.arange(m, device=dev)
            Lv[self.lay.r0 + i, i] = 1.0
            if self.d is not None:  # diag(LᵀAL) at L = I is diag(A): the diagonal entries of the local rows
                self.d.zero_()
                if isinstance(self.A, CsrRows):
                    self.d[self.lay.r0 + i] = self.A.diagonal()
                else:
                    self.d[self.lay.r0 + i] = self.A.view(n, m)[self.lay.r0 + i, i]
                if self.world > 1:
                    dist.all_reduce(self.d)
        else:
            self.L.copy_(l0_rows)
            if self.d is not None:
                self.refresh_diagonal()

    # ------------------------------------------------------------- helpers --
    def gather_l(self) -> torch.Tensor:
        """Full L (n×n column-major, flat) on every rank."""
        out = torch.empty(self.lay.n * self.lay.n, dtype=torch.float64, device=self.L.device)
        self._gather_panel(self.L, out)
        return out

    def refresh_diagonal(self):
        """Exact diag(LᵀAL) = Σ_p diag(L_pᵀ·(A_p·L)) (needs all of L: n² traffic)."""
        lay = self.lay
        n, m = lay.n, lay.m
        full = self.gather_l()
        AL = torch.empty(m * n, dtype=torch.float64, device=self.L.device)
        apply_rows(self.ops, self.A, n, full, n, n, AL, m)  # (A·L)[R_p, :] = A_p·L
        part = (AL.view(n, m) * self.L.view(n, m)).sum(dim=1)
        if self.world > 1:
            dist.all_reduce(part)
        self.d.copy_(part)

    def _probabilities(self) -> np.ndarray:  # adarbfgs.cpp:23-36 on the carried diagonal
        d = self.d.cpu().numpy()
        p = np.array([d[b[0]:b[-1] + 1].sum() for b in self.blocks])
        if p.min() <= 0.0:
            raise NumericalError("adaptive_block_probabilities: non-positive block trace; "
                                 "the factor has degenerated")
        return p / p.sum()

    # --------------------------------------------------------------- step --
    def step(self):
        lay, ops = self.lay, self.ops
        n, m = lay.n, lay.m
        p = self._probabilities() if self.rule == "cols" else None
        for _ in range(self.max_redraws + 1):
            if self.rule == "gauss":
                q = lay.q
                ops.sketch(self.St, n, q, n, self.seed, self.draw)
                self.draw += 1
                ops.gemm(m, q, n, self.L, m, False, self.St, n, True, self.Sp, m)            # S_p = L_p·S̃
            else:
                if self.rule == "cols":
                    cols = self.blocks[self.rng.categorical(p)]
                else:
                    cols = [int(v) for v in self.rng.uniform_subset(n, lay.q)]
                q = len(cols)
                h = self._idx_host[self._idx_slot, :q]
                self._idx_slot = (self._idx_slot + 1) % 4
                h.numpy()[:] = cols
                self.idx[:q].copy_(h, non_blocking=True)
                ops.gather_columns(self.L, m, m, self.idx, q, self.Sp)                        # S_p = L_p[:, C]
            self._all_gather_rows(self.Sp[: m * q], self.S[: n * q], q)                       # S
            apply_rows(ops, self.A, n, self.S, n, q, self.ASp, m)                                # (AS)_p = A_p·S
            G, Z = self.GZ[: q * q], self.GZ[q * q: q * q + q * n]
            ops.gemm(q, q, m, self.Sp, m, True, self.ASp, m, True, G, q)                       # S_pᵀ(AS)_p
            ops.gemm(q, n, m, self.ASp, m, True, self.L, m, True, Z, q)                        # (AS)_pᵀ L_p
            if self.world > 1:
                dist.all_reduce(self.GZ[: q * q + q * n])                                     # [G | Z]
            try:
                ops.ada_core(G, q, Z, n, None if self.rule == "gauss" else self.idx, self.St, self.T,
                             self.R, self.B, self.scratch)                                     # R, B = T − R·Z
            except GramRankDeficientError:
                self.redraws += 1  # G, Z identical on every rank: all ranks redraw together
                continue
            ops.gemm(m, q, q, self.Sp, m, False, self.R, q, True, self.SRp, m)                # (S·R)_p
            ops.gemm(m, n, q, self.SRp, m, False, self.B, q, True, self.L, m, 1.0, 1.0)      # L_p += (S·R)_p·B
            if self.d is not None:
                ops.pdiag_update(self.B, q, n, None, self.idx, self.d)                        # Eq. 8.2 diagonal
            self.k += 1
            return
        raise GramRankDeficientError("sketch rejection limit exceeded")

    def residual(self) -> float:
        """‖I − A·L·Lᵀ‖_F: X_p = L_p·Lᵀ from the gathered L, then the row-panel residual."""
        lay = self.lay
        n, m = lay.n, lay.m
        full = self.gather_l()
        Xp = torch.empty(m * n, dtype=torch.float64, device=self.L.device)
        self.ops.gemm(m, n, n, self.L, m, False, full, n, False, Xp, m)                       # X_p = L_p·Lᵀ
        part = self.ops.residual_rows_sq(self.prob, m, lay.r0, Xp, m)
        t = torch.tensor([part], dtype=torch.float64, device=self.L.device)
        if self.world > 1:
            dist.all_reduce(t)
        return float(t.item()) ** 0.5


def chunk_bounds(n: int, world: int):
    """2·world contiguous row chunks (sizes differ by at most one)."""
    return row_partition(n, 2 * world)


class SymmetricShardedRBFGS:
    """RBFGS with the upper triangle of X distributed over the ranks (SURVEY §8e,
    the symmetric-tile refinement of the row split).

    The rows are cut into 2P chunks; rank p owns chunks p and 2P−1−p, which
    balances the upper-triangular work (chunk c holds the trapezoid
    X[R_c, r0_c:n], the diagonal block stored in full).  Per iteration, with
    every product on the sm_100a engine through the device-pointer C ABI:

        Y_c      = A[R_c, :]·S                          local   2·m·n·q
        Y        = all-gather(Y_c)                      NCCL    n×q
        W       += X_c·Y[r0:]  and  X_c[:, m:]ᵀ·Y[R_c]   local   4·area·q
        W        = all-reduce(W partials)               NCCL    n×q
        P        = all-reduce(Σ_c Y[R_c]ᵀ·[S W][R_c])    NCCL    2q²
        M        = core(P)                              replicated
        V_c      = [S W][R_c]·M                         local
        X_c     += V_c·[S W][r0:]ᵀ   (diagonal block by K-SYMUPD, exactly symmetric)   2·area·2q

    Per-rank FLOPs ≈ 6n²q/P — the single-GPU count split evenly — against 8n²q/P
    for the full row panels of RowShardedRBFGS.
    """

    def __init__(self, ops, n: int, q: int, a_rows_of_chunk, *, seed: int = 0, prob: ProblemMatrix | None = None,
                 max_redraws: int = 100, device=None, deferred: bool | None = None):
        """a_rows_of_chunk(r0, r1) -> A[r0:r1, :] as a flat column-major (r1−r0)×n tensor or a
        CsrRows panel (sparse A, configs 4/5).

        deferred (default: when ops has core_async and SI_SHARD_SYNC_PD is unset): the PD test
        of SᵀAS is read one attempt late.  A rejected core leaves M = 0, so its update adds
        exact zeros and the attempt behind it is the redraw the synchronous loop would make;
        the draws, the accepted updates and the redraw accounting are those of the synchronous
        loop once finalize() has run (gather_x / residual call it)."""
        self.ops, self.n, self.q, self.seed, self.prob, self.max_redraws = ops, n, q, seed, prob, max_redraws
        if deferred is None:
            deferred = hasattr(ops, "core_async") and not os.environ.get("SI_SHARD_SYNC_PD") and max_redraws >= 1
        self.deferred = deferred
        self._pending = []        # (slot, event) of attempts whose PD status is not read yet
        self._consecutive = 0     # rejections since the last accepted attempt
        self._attempts = 0
        self._steps_done = 0      # step() calls returned
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.bounds = chunk_bounds(n, self.world)
        P = self.world
        self.chunks = [self.rank, 2 * P - 1 - self.rank]
        self.draw = 0
        self.redraws = 0
        A0 = a_rows_of_chunk(self.bounds[self.chunks[0]], self.bounds[self.chunks[0] + 1])
        dev = device if device is not None else (A0.val.device if isinstance(A0, CsrRows) else A0.device)
        f = dict(dtype=torch.float64, device=dev)
        self.A, self.X = {}, {}
        for c in self.chunks:
            r0, r1 = self.bounds[c], self.bounds[c + 1]
            self.A[c] = A0 if c == self.chunks[0] else a_rows_of_chunk(r0, r1)
            self.X[c] = torch.zeros((r1 - r0) * (n - r0), **f)
        self.S = torch.empty(n * q, **f)
        self.Y = torch.empty(n * q, **f)
        self.U = torch.empty(n * 2 * q, **f)  # [S W], column-major n×2q
        self.P = torch.empty(q * 2 * q, **f)
        self.M = torch.empty(4 * q * q, **f)
        mc = max(self.bounds[c + 1] - self.bounds[c] for c in range(2 * P))
        self.Yc = torch.empty(mc * q, **f)
        self.Vc = torch.empty(mc * 2 * q, **f)
        self.Uc = torch.empty(mc * 2 * q, **f)
        self.scratch = torch.empty(6 * q * q + 2 * q + 16, **f)
        self.gather = torch.empty(2 * P * mc * q, **f)
        # Y gather: each rank writes its two chunks' Y rows straight into send (2 × q × mc,
        # padding rows never read); the gathered (P, 2, q, mc) block goes to Y's rows in one
        # index_copy (src: valid gathered columns, dst: their global rows)
        self._mc = mc
        self.send = torch.zeros(2 * mc * q, **f)
        src, dst = [], []
        for p in range(P):
            for j, c in enumerate((p, 2 * P - 1 - p)):
                r0, r1 = self.bounds[c], self.bounds[c + 1]
                src.extend((p * 2 + j) * mc + i for i in range(r1 - r0))
                dst.extend(range(r0, r1))
        self._y_src = torch.tensor(src, dtype=torch.int64, device=dev)
        self._y_dst = torch.tensor(dst, dtype=torch.int64, device=dev)
        self._ring = 64
        self._status = torch.zeros(self._ring, dtype=torch.int32, device=dev)
        self._status_host = torch.zeros(self._ring, dtype=torch.int32,
                                        pin_memory=self._status.is_cuda)
        self.set_identity()

    def _m(self, c):
        return self.bounds[c + 1] - self.bounds[c]

    def set_identity(self):
        for c in self.chunks:
            m = self._m(c)
            xv = self.X[c].view(self.n - self.bounds[c], m)  # column-major m×(n−r0) == row-major (n−r0, m)
            xv.zero_()
            i = torch.arange(m, device=xv.device)
            xv[i, i] = 1.0

    def _rows(self, buf, ncols, r0, r1):
        """rows r0..r1 of a column-major n×ncols buffer, as an (ncols, r1−r0) view."""
        return buf.view(ncols, self.n)[:, r0:r1]

    def _all_gather_y(self):
        """Y (n×q) from the ranks' chunk rows (already in self.send); chunk sizes differ by at most one."""
        n, q, P, mc = self.n, self.q, self.world, self._mc
        if P > 1:
            dist.all_gather_into_tensor(self.gather, self.send)
            g = self.gather
        else:
            g = self.send
        cols = g.view(P * 2, q, mc).permute(1, 0, 2).reshape(q, P * 2 * mc)  # one copy
        self.Y.view(q, n).index_copy_(1, self._y_dst, cols.index_select(1, self._y_src))

    def step(self):
        """One accepted iteration (redraws included).  In the deferred mode the Gram status of
        this step's attempt is read during a later call, so a rejection-limit failure of step k
        raises GramRankDeficientError from step k+1 or from finalize() / gather_x() / residual()
        (the exception's `failed_step` attribute names k); the synchronous mode
        (SI_SHARD_SYNC_PD=1) raises from step k itself."""
        if not self.deferred:
            return self._step_sync()
        if self._consecutive:  # inside a rejection run: no speculation past the redraw limit
            self._settle(keep=0)
        self._attempt()
        self._settle(keep=1)
        self._steps_done += 1

    def finalize(self):
        """Read every outstanding PD status (redrawing for the rejected ones); may raise the
        rejection-limit error of an earlier step (see step())."""
        if self.deferred:
            self._settle(keep=0)

    def _attempt(self):
        slot = self._attempts % self._ring
        self._attempts += 1
        st = self._status[slot:slot + 1]
        self._one_attempt(lambda P, M: self.ops.core_async(P, self.q, self.q, M, self.scratch, st))
        self._status_host[slot:slot + 1].copy_(st, non_blocking=True)
        ev = None
        if st.is_cuda:
            ev = torch.cuda.Event()
            ev.record()
        self._pending.append((slot, ev))

    def _settle(self, keep: int):
        """Read the oldest statuses until at most `keep` attempts are outstanding.  A rejected
        attempt was a no-op (M = 0) and the attempt behind it is its redraw, so each rejection
        owes one more attempt; inside a rejection run the attempts are read one at a time."""
        owed = 0
        while self._pending and (len(self._pending) > keep or owed or self._consecutive):
            slot, ev = self._pending.pop(0)
            if ev is not None:
                ev.synchronize()
            if int(self._status_host[slot]) == 0:
                self._consecutive = 0
            else:
                self.redraws += 1
                self._consecutive += 1
                if self._consecutive > self.max_redraws:
                    self._consecutive = 0
                    err = GramRankDeficientError("sketch rejection limit exceeded")
                    err.failed_step = self._steps_done  # 1-based: the step whose draws ran out
                    raise err
                owed += 1
            if not self._pending and owed:
                owed -= 1
                self._attempt()

    def _step_sync(self):
        for _ in range(self.max_redraws + 1):
            try:
                self._one_attempt(lambda P, M: self.ops.core(P, self.q, self.q, M, self.scratch))
            except GramRankDeficientError:
                self.redraws += 1
                continue
            return
        raise GramRankDeficientError("sketch rejection limit exceeded")

    def _one_attempt(self, core):
        n, q, ops = self.n, self.q, self.ops
        S, W = self.U[: n * q], self.U[n * q:]
        ops.sketch(S, n, q, n, self.seed, self.draw)
        self.draw += 1
        # Y rows of the owned chunks, then the full Y
        for j, c in enumerate(self.chunks):
            apply_rows(ops, self.A[c], n, S, n, q, self.send[j * q * self._mc:], self._mc)
        self._all_gather_y()
        # W = X·Y from the upper trapezoids: X_c·Y[r0:] and the strictly-upper part transposed
        W.zero_()
        for c in self.chunks:
            r0, m = self.bounds[c], self._m(c)
            r1 = r0 + m
            ops.gemm(m, q, n - r0, self.X[c], m, False, self.Y[r0:], n, True, W[r0:], n, 1.0, 1.0)
            if r1 < n:
                ops.gemm(n - r1, q, m, self.X[c][m * m:], m, True, self.Y[r0:], n, True, W[r1:], n, 1.0, 1.0)
        if self.world > 1:
            dist.all_reduce(W)
        # P = Yᵀ·[S W] over the owned rows, all-reduced
        for j, c in enumerate(self.chunks):  # the first chunk overwrites P (beta = 0)
            r0, m = self.bounds[c], self._m(c)
            ops.gemm(q, 2 * q, m, self.Y[r0:], n, True, self.U[r0:], n, True, self.P, q, 1.0, float(j > 0))
        if self.world > 1:
            dist.all_reduce(self.P)
        core(self.P, self.M)
        for c in self.chunks:
            r0, m = self.bounds[c], self._m(c)
            r1 = r0 + m
            # V_c = U[R_c]·M (m×2q); the diagonal block by K-SYMUPD, the rest by one GEMM
            ops.gemm(m, 2 * q, 2 * q, self.U[r0:], n, False, self.M, 2 * q, True, self.Vc, m)
            ops.symupd(m, 2 * q, self.Vc, m, self.U[r0:], n, self.X[c], m)
            if r1 < n:
                ops.gemm(m, n - r1, 2 * q, self.Vc, m, False, self.U[r1:], n, False, self.X[c][m * m:], m,
                         1.0, 1.0)

    def gather_x(self) -> torch.Tensor:
        """Full X (n×n column-major, flat) on every rank (tests / export / residual)."""
        self.finalize()
        n = self.n
        full = torch.zeros(n * n, dtype=torch.float64, device=self.X[self.chunks[0]].device)
        fv = full.view(n, n)  # fv[j, i] = X(i, j)
        for c in self.chunks:
            r0, m = self.bounds[c], self._m(c)
            xv = self.X[c].view(n - r0, m)  # xv[j', i'] = X(r0 + i', r0 + j')
            fv[r0:, r0:r0 + m].copy_(xv)          # X(rows, cols ≥ r0)
            fv[r0:r0 + m, r0:].copy_(xv.t())      # mirror: X(cols, rows)
        if self.world > 1:  # every entry is written by exactly one rank (its chunk's owner)
            dist.all_reduce(full)
        return full

    def residual(self) -> float:
        """‖I − X·A‖_F (= ‖I − A·X‖_F) over the owned chunks' rows of the gathered X."""
        n = self.n
        full = self.gather_x()
        part = 0.0
        for c in self.chunks:
            r0, m = self.bounds[c], self._m(c)
            part += self.ops.residual_rows_sq(self.prob, m, r0, full[r0:], n)
        t = torch.tensor([part], dtype=torch.float64, device=full.device)
        if self.world > 1:
            dist.all_reduce(t)
        return float(t.item()) ** 0.5
