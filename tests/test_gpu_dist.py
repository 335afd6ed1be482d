"""GPU checks of the device-pointer C ABI and the row-sharded driver at world
size 1 (the only GPU count available to this run; N > 1 is covered on CPU by
tests/test_dist_cpu.py with the same driver code)."""
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


@pytest.mark.parametrize("ak,bk", [(False, True), (True, True), (False, False)])
@pytest.mark.parametrize("M,N,K", [(33, 17, 65), (256, 128, 512), (130, 256, 2048)])
def test_gemm_device_layouts(env, ak, bk, M, N, K):
    si, torch, ctx, ops = env
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K))
    b = rng.standard_normal((K, N))
    c0 = rng.standard_normal((M, N))
    A = torch.from_numpy((a if ak else a.T).copy().reshape(-1)).cuda()  # kmajor: row-major M×K
    B = torch.from_numpy((b.T if bk else b).copy().reshape(-1)).cuda()  # kmajor: col-major K×N
    Cm = torch.from_numpy(c0.T.copy().reshape(-1)).cuda()
    ops.gemm(M, N, K, A, K if ak else M, ak, B, K if bk else N, bk, Cm, M, 0.5, 2.0)
    torch.cuda.synchronize()
    got = Cm.cpu().numpy().reshape((N, M)).T
    ref = 0.5 * a @ b + 2.0 * c0
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max() * K


def test_sketch_deterministic_and_gaussian(env):
    si, torch, ctx, ops = env
    n, q = 4096, 64
    s1 = torch.empty(n * q, dtype=torch.float64, device="cuda")
    s2 = torch.empty_like(s1)
    ops.sketch(s1, n, q, n, 11, 3)
    ops.sketch(s2, n, q, n, 11, 3)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2)
    ops.sketch(s2, n, q, n, 11, 4)
    v = s2.cpu().numpy()
    assert abs(v.mean()) < 5e-3 and abs(v.std() - 1.0) < 5e-3
    assert not torch.equal(s1, s2)


def test_row_sharded_world1_matches_solver(env):
    si, torch, ctx, ops = env
    from paper_1602_01768_b200 import generators as G
    from paper_1602_01768_b200.dist import RowShardedRBFGS

    n, q, iters, seed = 512, 16, 15, 7
    a = G.config1_dense(n, seed=2)
    prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
    a_rows = torch.from_numpy(a.reshape(-1, order="F").copy()).cuda()
    sh = RowShardedRBFGS(ops, n, q, a_rows, seed=seed, prob=prob)
    for _ in range(iters):
        sh.step()
    x_sh = sh.gather_x().cpu().numpy().reshape((n, n), order="F")
    sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=seed)
    sol.step(iters)
    x_so = sol.iterate()
    assert np.linalg.norm(x_sh - x_so) / np.linalg.norm(x_so) <= 1e-9
    assert sh.residual() == pytest.approx(sol.residual(), rel=1e-9)


@pytest.mark.parametrize("rule", ["cols", "uniform", "gauss"])
def test_row_sharded_ada_world1(env, rule):
    """The sharded AdaRBFGS driver at world size 1 on the GPU against the oracle
    on the same index / sketch sequence, and its carried Eq. 8.2 diagonal against
    the exact diag(LᵀAL)."""
    si, torch, ctx, ops = env
    from oracle import oracle as O
    from paper_1602_01768_b200.dist import RowShardedAdaRBFGS

    n, q, iters, seed = 300, 20, 40, 6
    rng = O.RngStream(41)
    b = rng.gaussian_matrix(n, n)
    a = np.asfortranarray(b @ b.T / n + np.eye(n))
    prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
    a_rows = torch.from_numpy(a.reshape(-1, order="F").copy()).cuda()
    sh = RowShardedAdaRBFGS(ops, n, q, a_rows, rule=rule, seed=seed, prob=prob)
    sketches = []
    for _ in range(iters):
        sh.step()
        if rule == "gauss":
            sketches.append(sh.St.cpu().numpy().reshape((n, q), order="F").copy())
    lf = sh.gather_l().cpu().numpy().reshape((n, n), order="F")
    if rule == "gauss":
        ref = np.eye(n)
        for s in sketches:
            ref = O.adarbfgs_update_factor(ref, a, s)
    else:
        ref = O.run_adarbfgs(a, q, rule=O.ADA_COLS if rule == "cols" else O.ADA_COLS_UNIFORM, tol=0.0,
                             max_iters=iters, every_k=iters, seed=seed).x
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) <= 1e-9
    assert sh.residual() == pytest.approx(np.linalg.norm(np.eye(n) - a @ lf @ lf.T), rel=1e-8)
    if rule == "cols":
        d = sh.d.cpu().numpy()
        assert np.allclose(d, np.einsum("ij,ij->j", lf, a @ lf), rtol=1e-10, atol=0)


def test_symmetric_sharded_world1_matches_solver(env):
    si, torch, ctx, ops = env
    from paper_1602_01768_b200 import generators as G
    from paper_1602_01768_b200.dist import SymmetricShardedRBFGS

    n, q, iters, seed = 600, 24, 12, 3  # odd chunk offsets exercise the unaligned (non-TMA) operands
    a = G.config1_dense(n, seed=4)
    prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def rows(r0, r1):
        return at[:, r0:r1].contiguous().reshape(-1)

    sh = SymmetricShardedRBFGS(ops, n, q, rows, seed=seed, prob=prob)
    for _ in range(iters):
        sh.step()
    x_sh = sh.gather_x().cpu().numpy().reshape((n, n), order="F")
    sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=seed)
    sol.step(iters)
    x_so = sol.iterate()
    assert np.linalg.norm(x_sh - x_so) / np.linalg.norm(x_so) <= 1e-9
    assert np.array_equal(x_sh, x_sh.T)
    assert sh.residual() == pytest.approx(sol.residual(), rel=1e-9)


def test_sharded_drivers_with_csr_panels_world1(env):
    """Sparse A through the sharded drivers' CSR row panels (si_spmm_csr_device):
    the symmetric-chunk RBFGS driver against the single-GPU solver on the same CSR
    problem, and the row-sharded AdaRBFGS driver against the oracle."""
    si, torch, ctx, ops = env
    from oracle import oracle as O
    from paper_1602_01768_b200 import generators as G
    from paper_1602_01768_b200.dist import CsrRows, RowShardedAdaRBFGS, SymmetricShardedRBFGS

    n, q, iters = 1024, 32, 10
    rowptr, colind, val = G.config5_csr(n, half_bandwidth=16, seed=1)
    prob = si.ProblemMatrix(csr=(rowptr, colind, val), n=n, symmetry=si.Symmetry.spd, context=ctx)
    sh = SymmetricShardedRBFGS(ops, n, q, lambda r0, r1: CsrRows.from_host(rowptr, colind, val, r0, r1, "cuda"),
                               seed=4)
    for _ in range(iters):
        sh.step()
    x_sh = sh.gather_x().cpu().numpy().reshape((n, n), order="F")
    sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=4)
    sol.step(iters)
    x_so = sol.iterate()
    assert np.linalg.norm(x_sh - x_so) / np.linalg.norm(x_so) <= 1e-9
    assert np.array_equal(x_sh, x_sh.T)

    a = prob.data()
    ada = RowShardedAdaRBFGS(ops, n, 16, CsrRows.from_host(rowptr, colind, val, 0, n, "cuda"), rule="cols", seed=2)
    for _ in range(12):
        ada.step()
    lf = ada.gather_l().cpu().numpy().reshape((n, n), order="F")
    ref = O.run_adarbfgs(a, 16, rule=O.ADA_COLS, tol=0.0, max_iters=12, every_k=12, seed=2).x
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) <= 1e-9


@pytest.mark.parametrize("max_redraws", [100, 1])
def test_symmetric_deferred_pd_check_gpu(env, max_redraws):
    """si_rbfgs_core_device_async + the deferred status read against the synchronous loop
    on an indefinite A (44 of 96 eigenvalues negative), so that many Gaussian draws give a non-PD
    SᵀAS: identical X, draw count and redraw count (and the same error at a tight limit)."""
    si, torch, ctx, ops = env
    from paper_1602_01768_b200.api import GramRankDeficientError
    from paper_1602_01768_b200.dist import SymmetricShardedRBFGS

    n, q, iters, seed = 96, 2, 16, 11
    rng = np.random.default_rng(0)
    qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([np.linspace(0.5, 1.5, 52), -np.linspace(0.5, 1.5, n - 52)])
    a = (qm * lam) @ qm.T
    a = 0.5 * (a + a.T)
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def rows(r0, r1):
        return at[:, r0:r1].contiguous().reshape(-1)

    def run(deferred):
        sh = SymmetricShardedRBFGS(ops, n, q, rows, seed=seed, max_redraws=max_redraws, deferred=deferred)
        err = False
        try:
            for _ in range(iters):
                sh.step()
            sh.finalize()
        except GramRankDeficientError:
            err = True
        return sh.gather_x().cpu().numpy(), sh.draw, sh.redraws, err

    xs, ds, rs, es = run(False)
    xd, dd, rd, ed = run(True)
    if max_redraws == 100:
        assert rs > 0 and not es  # the problem does exercise rejections
    assert (dd, rd, ed) == (ds, rs, es)
    assert np.array_equal(xd, xs)
