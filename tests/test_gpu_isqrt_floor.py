"""The reference's inverse-square-root rejection contract on the GPU path.

sym_inv_sqrt (proj/src/linalg.cpp:144-155) throws iff an eigenvalue
λ ≤ 1e-14·λmax or λ ≤ 0; run_adarbfgs redraws on that throw
(proj/src/adarbfgs.cpp:145-155).  The GPU keeps Newton–Schulz's root only when it
certifies λmin/λmax > 1e-12 and otherwise decides with the reference's Jacobi
and floor (kernels_small.cuh jacobi_isqrt_block), so accept / reject — and with it
every later draw — follows the oracle.  Covered: the fused one-CTA path (q ≤ 64)
and the GEMM-engine path (q > 64), Grams with λmin/λmax on both sides of the
floor, and a 200-iteration AdaRBFGS run whose early sketches hit the floor.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

FLOOR = 1e-14


@pytest.fixture(scope="module")
def si():
    import paper_1602_01768_b200 as si

    return si


def spectrum_matrix(q, ratio, seed):
    """M = Q·diag(λ)·Qᵀ, λ log-spaced from `ratio` to 1, Q orthogonal (numpy QR of an
    RngStream Gaussian)."""
    g = O.RngStream(seed).gaussian_matrix(q, q)
    qm, _ = np.linalg.qr(g)
    lam = np.logspace(np.log10(ratio), 0.0, q)
    m = (qm * lam) @ qm.T
    return np.asfortranarray(0.5 * (m + m.T))


def oracle_decision(m):
    vals, _ = O.jacobi_eigendecomposition(m)
    ratio = vals.min() / vals.max()
    try:
        r = O.sym_inv_sqrt(m)
        return True, r, ratio
    except O.NumericalError:
        return False, None, ratio


@pytest.mark.parametrize("q", [8, 16, 48, 64, 96, 128, 256])
@pytest.mark.parametrize("ratio", [5e-15, 2e-14, 1e-13, 1e-9, 1e-3])
def test_floor_decision_matches_oracle(si, q, ratio):
    m = spectrum_matrix(q, ratio, seed=int(q * 7 + ratio * 1e15) % 100003)
    ok_ref, r_ref, got_ratio = oracle_decision(m)
    # the constructed spectrum survives rounding well away from the floor
    assert got_ratio <= 0.6 * FLOOR or got_ratio >= 1.5 * FLOOR, got_ratio
    if ok_ref:
        r = si.sym_inv_sqrt(m)
        kappa = 1.0 / max(got_ratio, 1e-300)
        # the unique symmetric root, equal to rounding: a perturbation of M of eps·‖M‖ moves
        # λmin^{-1/2} by ≈ κ·eps/2 relative, in either implementation
        assert np.linalg.norm(r - r_ref) <= 1e-13 * max(1e3, kappa) * np.linalg.norm(r_ref)
        assert np.array_equal(r, r.T) or np.linalg.norm(r - r.T) <= 1e-15 * np.linalg.norm(r)
    else:
        with pytest.raises(si.NumericalError):
            si.sym_inv_sqrt(m)


def test_floor_zero_and_indefinite(si):
    with pytest.raises(si.NumericalError):
        si.sym_inv_sqrt(np.zeros((5, 5)))
    with pytest.raises(si.NumericalError):
        si.sym_inv_sqrt(np.diag([1.0, 2.0, -1e-3]))
    for q in (8, 80):  # semidefinite: an exact zero eigenvalue
        v = O.RngStream(q).gaussian_matrix(q, q - 1)
        with pytest.raises(si.NumericalError):
            si.sym_inv_sqrt(v @ v.T)


def near_singular_problem(n, seed, bad_every=1):
    """A = Π·blockdiag([[1, 1−δ_k], [1−δ_k, 1]])·Πᵀ: 2×2 blocks with eigenvalues δ_k and 2 − δ_k,
    so a Gram holding both coordinates of a pair has λmin/λmax ≈ δ_k/2 — from 1e-15 (below the
    1e-14 floor) to 1e-10 — while A's own LLT pivots (1 and ≈ 2δ_k) stay clear of rounding;
    the pairs are scattered by a seeded permutation Π (so contiguous blocks mix them)."""
    deltas = [2e-15, 1e-14, 6e-14, 2e-13, 2e-10, 0.5, 0.2, 1.0]
    a = np.zeros((n, n))
    for k in range(n // 2):
        d = deltas[k % len(deltas)] if k % bad_every == 0 else 0.7
        i, j = 2 * k, 2 * k + 1
        a[i, i] = a[j, j] = 1.0
        a[i, j] = a[j, i] = 1.0 - d
    if n % 2:
        a[n - 1, n - 1] = 1.0
    rng = O.RngStream(seed)
    perm = np.argsort([rng.uniform() for _ in range(n)], kind="stable")
    return np.asfortranarray(a[np.ix_(perm, perm)])


@pytest.mark.parametrize("sampler,q", [("uniform", 4), ("cols", 2), ("uniform", 80)])
def test_adarbfgs_near_singular_draws_match_oracle(si, sampler, q):
    """200 iterations (uniform q=4, Eq. 8.2 blocks q=2) over sketches that start out
    near-singular: every executed draw (rejected ones included) equals the oracle's and
    the factor matches.  q = 80 runs the GEMM-engine Newton–Schulz + Jacobi fallback."""
    n, iters = (32, 200) if q < 64 else (160, 60)
    a = near_singular_problem(n, seed=7 + q, bad_every=1 if q < 64 else 20)
    orule = O.ADA_COLS_UNIFORM if sampler == "uniform" else O.ADA_COLS
    ref = O.run_adarbfgs(a, q, rule=orule, tol=0.0, max_iters=iters, every_k=20, seed=11, max_redraws=1000,
                         max_outcomes=iters * q * 50)
    ctx = si.Context(0)
    ctx.set_draw_log(iters * q * 50)
    rule = si.SketchRule.adaptive_cols_uniform(q) if sampler == "uniform" else si.SketchRule.adaptive_cols(n, q)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd, context=ctx), rule, tol=0.0,
                                       max_iters=iters, seed=11, max_redraws=1000,
                                       track=si.TrackOptions(residual_every_k=20)))
    drawn = ctx.draw_log()
    per = q if sampler == "uniform" else 1
    print(f"{sampler} q={q}: {drawn.size // per} draws for {iters} iterations, redraws {res.state.redraws}")
    assert res.state.redraws > 0  # the floor was hit
    assert np.array_equal(drawn, ref.outcomes[:drawn.size])
    assert drawn.size == iters * per + res.state.redraws * per
    assert res.state.k == ref.k == iters
    err = np.linalg.norm(res.state.l - ref.x) / np.linalg.norm(ref.x)
    print(f"  factor rel err {err:.3e}")
    assert err <= 1e-6
