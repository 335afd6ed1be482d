"""Parity at BASELINE.json's full sizes through size-independent properties
(the oracle cannot run n = 16384 … 98304 in seconds).

One update at full size with a known sketch must satisfy the quasi-Newton
secant equation exactly (up to rounding): X⁺·(A·S) = S for RBFGS (Eq. 7.17:
X⁺ = P + (I − PA)X(I − AP) with PAS = S), and L⁺L⁺ᵀ·(A·S) = S for AdaRBFGS
with S = L·S̃ (adarbfgs.cpp:12-21; the factored iterate is the BFGS update of
LLᵀ).  The RBFGS iterate must also be exactly symmetric.  Configs 3, 4 and 5
(SURVEY §8d), first iteration from X₀ = I / L₀ = I.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_1602_01768_b200 as si
    from paper_1602_01768_b200.dist import CudaPanelOps

    ctx = si.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    return si, torch, ctx, CudaPanelOps(ctx)


def _device_view(torch, ptr, numel):
    """A float64 CUDA tensor over a library-owned device buffer (no copy)."""

    class _Holder:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (p, False), "version": 3}

    return torch.as_tensor(_Holder(ptr, numel), device="cuda")


def _secant_residual(torch, ops, x_ptr, n, ay, s):
    """‖X·(AS) − S‖_F / ‖S‖_F with X the library's device iterate (column-major n×n)."""
    q = s.shape[1]
    X = _device_view(torch, x_ptr, n * n)
    AY = torch.from_numpy(np.asfortranarray(ay).reshape(-1, order="F").copy()).cuda() if isinstance(ay, np.ndarray) \
        else ay
    out = torch.empty(n * q, dtype=torch.float64, device="cuda")
    ops.gemm(n, q, n, X, n, False, AY, n, True, out, n)
    torch.cuda.synchronize()
    S = torch.from_numpy(np.asfortranarray(s).reshape(-1, order="F").copy()).cuda()
    return float(torch.linalg.norm(out - S) / torch.linalg.norm(S))


def test_config3_rbfgs_secant_and_symmetry(env):
    si, torch, ctx, ops = env
    from paper_1602_01768_b200 import generators as G

    n, q = 16384, 128
    a_dev = G.config3_dense_device(n, seed=0)  # row-major tensor of the symmetric A
    prob = si.ProblemMatrix(a_dev.cpu().numpy(), si.Symmetry.spd, context=ctx)
    del a_dev
    torch.cuda.empty_cache()
    sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian(q), seed=0)
    s = si.RngStream(3).gaussian_matrix(n, q)
    sol.step_with_sketch(s=s)
    A = _device_view(torch, si._lib.load().si_problem_dense_device(prob.handle), n * n)
    S = torch.from_numpy(np.asfortranarray(s).reshape(-1, order="F").copy()).cuda()
    AS = torch.empty(n * q, dtype=torch.float64, device="cuda")
    ops.gemm(n, q, n, A, n, False, S, n, True, AS, n)
    assert _secant_residual(torch, ops, sol.iterate_device_ptr(), n, AS, s) <= 1e-10
    X = _device_view(torch, sol.iterate_device_ptr(), n * n).view(n, n)
    assert torch.equal(X, X.t())  # exactly symmetric (mirrored upper tiles)
    # a second update keeps both properties for the new sketch
    s2 = si.RngStream(4).gaussian_matrix(n, q)
    sol.step_with_sketch(s=s2)
    S2 = torch.from_numpy(np.asfortranarray(s2).reshape(-1, order="F").copy()).cuda()
    ops.gemm(n, q, n, A, n, False, S2, n, True, AS, n)
    assert _secant_residual(torch, ops, sol.iterate_device_ptr(), n, AS, s2) <= 1e-10
    assert torch.equal(X, X.t())


def test_config4_adarbfgs_factored_secant(env):
    si, torch, ctx, ops = env
    from paper_1602_01768_b200 import generators as G

    n, q = 65536, 256
    rowptr, colind, val = G.config4_csr(n)
    prob = si.ProblemMatrix(csr=(rowptr, colind, val), n=n, symmetry=si.Symmetry.spd, context=ctx)
    sol = si.Solver(prob, si.Method.adarbfgs, si.SketchRule.adaptive_cols_uniform(q), seed=0)
    idx = np.sort(si.RngStream(5).uniform_subset(n, q))
    sol.step_with_sketch(idx=idx)
    # L₀ = I: S = L₀·S̃ = I[:, idx]; A·S = A[:, idx] (= rows idx of the symmetric A)
    a_cols = np.zeros((n, q))
    for j, r in enumerate(idx):
        a_cols[colind[rowptr[r]:rowptr[r + 1]], j] = val[rowptr[r]:rowptr[r + 1]]
    s = np.zeros((n, q))
    s[idx, np.arange(q)] = 1.0
    Lp = _device_view(torch, sol.iterate_device_ptr(), n * n)
    AS = torch.from_numpy(np.asfortranarray(a_cols).reshape(-1, order="F").copy()).cuda()
    t = torch.empty(n * q, dtype=torch.float64, device="cuda")
    out = torch.empty(n * q, dtype=torch.float64, device="cuda")
    ops.gemm(n, q, n, Lp, n, True, AS, n, True, t, n)     # L⁺ᵀ·(AS)
    ops.gemm(n, q, n, Lp, n, False, t, n, True, out, n)   # L⁺·(L⁺ᵀ·AS)
    torch.cuda.synchronize()
    S = torch.from_numpy(np.asfortranarray(s).reshape(-1, order="F").copy()).cuda()
    assert float(torch.linalg.norm(out - S) / torch.linalg.norm(S)) <= 1e-10


def test_config5_rbfgs_sparse_secant(env):
    si, torch, ctx, ops = env
    import scipy.sparse as sp

    from paper_1602_01768_b200 import generators as G

    n, q = 98304, 512
    rowptr, colind, val = G.config5_csr(n, half_bandwidth=64, seed=0)
    prob = si.ProblemMatrix(csr=(rowptr, colind, val), n=n, symmetry=si.Symmetry.spd, context=ctx)
    sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian(q), seed=0)
    s = si.RngStream(6).gaussian_matrix(n, q)
    sol.step_with_sketch(s=s)
    a = sp.csr_matrix((val, colind, rowptr), shape=(n, n))
    assert _secant_residual(torch, ops, sol.iterate_device_ptr(), n, np.asarray(a @ s), s) <= 1e-10
