"""GPU checks of the round-2 kernel paths through the device-pointer C ABI: the C-panel
update with the bulk-copy epilogue (short-K C += A·B: ragged tiles, every operand layout),
the row-blocked CSR SpMM (block sizes, ragged row counts, unsorted and duplicate column
indices — bitwise against a per-row reference order), K-SYMUPD over ragged sizes, and the
left-looking validate_spd decisions (first / last panel failures, n not a multiple of 128)."""
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


# K <= 256, M, N > 64, alpha = 1, beta != 0: the C-panel kernels (gemm_tma_cbulk_kernel for even M)
@pytest.mark.parametrize("ak,bk", [(False, True), (False, False), (True, True)])
@pytest.mark.parametrize("M,N,K", [(512, 256, 64), (300, 130, 64), (1026, 190, 32), (640, 448, 256), (258, 66, 16),
                                   (301, 130, 64), (770, 322, 40), (4100, 260, 8), (20000, 70, 64), (140, 9000, 48)])
def test_cpanel_update_shapes(env, ak, bk, M, N, K):
    si, torch, ctx, ops = env
    rng = np.random.default_rng(7 * M + N + K)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N))
    c0 = rng.standard_normal((M, N))
    A = torch.from_numpy((a if ak else a.T).copy().reshape(-1)).cuda()
    B = torch.from_numpy((b.T if bk else b).copy().reshape(-1)).cuda()
    for beta in (1.0, -0.5):
        Cm = torch.from_numpy(c0.T.copy().reshape(-1)).cuda()
        ops.gemm(M, N, K, A, K if ak else M, ak, B, K if bk else N, bk, Cm, M, 1.0, beta)
        torch.cuda.synchronize()
        got = Cm.cpu().numpy().reshape((N, M)).T
        ref = a @ b + beta * c0
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max() * K


@pytest.mark.parametrize("M,N,K,pad", [(300, 130, 64, 6), (512, 192, 128, 2), (258, 66, 32, 10)])
def test_cpanel_update_guard_bands(env, M, N, K, pad):
    # C with a leading dimension larger than M inside a sentinel-filled buffer: the bulk copies
    # must write exactly the M rows of each column — not the padding rows, nothing before or after
    si, torch, ctx, ops = env
    rng = np.random.default_rng(M + N + K + pad)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N))
    c0 = rng.standard_normal((M, N))
    ldc, guard, sentinel = M + pad, 4096, -7.25
    A = torch.from_numpy(a.T.copy().reshape(-1)).cuda()
    B = torch.from_numpy(b.T.copy().reshape(-1)).cuda()
    buf = torch.full((guard + ldc * N + guard,), sentinel, dtype=torch.float64, device="cuda")
    view = buf[guard:guard + ldc * N].view(N, ldc)
    view[:, :M] = torch.from_numpy(c0.T.copy()).cuda()
    ops.gemm(M, N, K, A, M, False, B, K, True, buf[guard:], ldc, 1.0, 1.0)
    torch.cuda.synchronize()
    out = buf.cpu().numpy()
    assert (out[:guard] == sentinel).all() and (out[guard + ldc * N:] == sentinel).all()
    body = out[guard:guard + ldc * N].reshape((N, ldc))
    assert (body[:, M:] == sentinel).all()
    ref = a @ b + c0
    assert np.abs(body[:, :M].T - ref).max() <= 1e-13 * np.abs(ref).max() * K


def test_cpanel_update_many_tiles_per_cta(env):
    # more work items than SMs: every CTA walks several tiles (C-in / C-out buffer reuse)
    si, torch, ctx, ops = env
    M, N, K = 4096, 2048, 64
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g)  # column-major M×K
    B = torch.randn(N, K, dtype=torch.float64, device="cuda", generator=g)  # K-major: column-major K×N
    C0 = torch.randn(N, M, dtype=torch.float64, device="cuda", generator=g)
    Cm = C0.clone()
    ops.gemm(M, N, K, A, M, False, B, K, True, Cm, M, 1.0, 1.0)
    torch.cuda.synchronize()
    ref = C0 + B @ A  # (N×K)·(K×M) = (A_cm·B_cm)ᵀ in row-major
    assert (Cm - ref).abs().max().item() <= 1e-12 * ref.abs().max().item()


def _csr_reference(rowptr, colind, val, P):
    # per-row sums in storage order (what both SpMM kernels compute, FMA rounding aside)
    n = len(rowptr) - 1
    out = np.zeros((n, P.shape[1]))
    for i in range(n):
        for t in range(rowptr[i], rowptr[i + 1]):
            out[i] += val[t] * P[colind[t]]
    return out


@pytest.mark.parametrize("n,k", [(257, 64), (300, 128), (515, 192), (1024, 256), (999, 512), (130, 96)])
@pytest.mark.parametrize("kind", ["banded", "random_unsorted", "duplicates_and_empty"])
def test_spmm_rowblock(env, n, k, kind):
    si, torch, ctx, ops = env
    rng = np.random.default_rng(n + k)
    rows = []
    for i in range(n):
        if kind == "banded":
            cols = np.arange(max(0, i - 9), min(n, i + 10))
        elif kind == "random_unsorted":
            cols = rng.permutation(n)[: rng.integers(1, 24)]
        else:
            cols = rng.integers(0, n, size=rng.integers(0, 12)) if i % 5 else np.zeros(0, dtype=np.int64)
            if len(cols) > 2:
                cols[1] = cols[0]  # a duplicate column inside the row
        rows.append(np.asarray(cols, dtype=np.int64))
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    colind = np.concatenate(rows).astype(np.int32) if rowptr[-1] else np.zeros(0, dtype=np.int32)
    val = rng.standard_normal(int(rowptr[-1]))
    P = rng.standard_normal((n, k))
    rp, ci, va = (torch.from_numpy(x).cuda() for x in (rowptr, colind, val))
    Pd = torch.from_numpy(P.T.copy().reshape(-1)).cuda()  # column-major n×k
    guard = 1024
    buf = torch.full((guard + k * n + guard,), np.nan, dtype=torch.float64, device="cuda")
    buf[:guard] = -7.25
    buf[guard + k * n:] = -7.25
    Y = buf[guard:guard + k * n]
    ops.spmm(n, n, rp, ci, va, Pd, n, k, Y, n)
    torch.cuda.synchronize()
    assert (buf[:guard] == -7.25).all().item() and (buf[guard + k * n:] == -7.25).all().item()
    got = Y.cpu().numpy().reshape((k, n)).T
    ref = _csr_reference(rowptr, colind, val, P)
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max()) * 32


@pytest.mark.parametrize("n,q", [(1280, 64), (2100, 40), (2500, 128), (4000, 16)])
def test_symupd_shapes(env, n, q):
    si, torch, ctx, ops = env
    g = torch.Generator(device="cuda").manual_seed(n + q)
    X0 = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    X0 = X0 + X0.T
    V = torch.randn(2 * q, n, dtype=torch.float64, device="cuda", generator=g) * 1e-2  # column-major n×2q
    U = torch.randn(2 * q, n, dtype=torch.float64, device="cuda", generator=g) * 1e-2
    X = X0.clone()
    ops.symupd(n, 2 * q, V, n, U, n, X, n)
    torch.cuda.synchronize()
    ref = X0.T + V.T @ U  # column-major X(r, c) = X.T[r, c]
    up = torch.triu(ref)
    ref = up + torch.triu(up, 1).T
    assert (X.T - ref).abs().max().item() <= 1e-13 * ref.abs().max().item()
    assert torch.equal(X, X.T)  # exactly symmetric: upper tiles mirrored


@pytest.mark.parametrize("n", [64, 128, 129, 300, 1000, 1409])
def test_validate_spd_decisions(env, n):
    si, torch, ctx, ops = env
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    a = b @ b.T / n + 0.5 * np.eye(n)
    cases = {
        "spd": (a, True),
        "first_pivot": (a - np.diag([2.0 * a[0, 0]] + [0.0] * (n - 1)), False),
        "last_pivot": (a - np.diag([0.0] * (n - 1) + [50.0]), False),
        "middle_pivot": (a - np.diag([0.0] * (n // 2) + [50.0] + [0.0] * (n - n // 2 - 1)), False),
        "semidefinite": (np.ones((n, n)), False),
    }
    for name, (m, ok) in cases.items():
        assert (np.linalg.eigvalsh(m).min() > 0) == ok, name
        p = si.ProblemMatrix(np.asfortranarray(m), si.Symmetry.spd, context=ctx)
        if ok:
            p.validate_spd()
        else:
            with pytest.raises(Exception) as ei:
                p.validate_spd()
            assert "Cholesky failed" in str(ei.value), name


def test_validate_spd_near_singular_matches_llt(env):
    # the decision is the LLT's: a pivot that the elimination drives to ≤ 0 (here through
    # cancellation in a late Schur complement), not an eigenvalue estimate
    si, torch, ctx, ops = env
    n = 520
    rng = np.random.default_rng(5)
    u = rng.standard_normal((n, 3))
    for shift, ok in ((1e-3, True), (-1e-3, False)):
        m = u @ u.T + np.eye(n)
        m[-1, -1] = m[-1, :-1] @ np.linalg.solve(m[:-1, :-1], m[:-1, -1]) + shift  # last Schur pivot = shift
        try:
            np.linalg.cholesky(m)
            llt_ok = True
        except np.linalg.LinAlgError:
            llt_ok = False
        assert llt_ok == ok
        p = si.ProblemMatrix(np.asfortranarray(m), si.Symmetry.spd, context=ctx)
        if ok:
            p.validate_spd()
        else:
            with pytest.raises(Exception):
                p.validate_spd()
