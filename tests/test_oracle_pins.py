"""Pin the CPU oracle to the reference's own known-answer tests (SURVEY §4 pin table).

Each test restates one reference test case (file:line cited) against the oracle
restatement in oracle/stochinv_oracle.cpp.  These run without a GPU.
"""
import numpy as np
import pytest

from oracle import oracle as O


def fixture_a():
    return np.array([[2.0, 1.0], [1.0, 2.0]], order="F")


def coordinate_sketch(n, idx):
    s = np.zeros((n, len(idx)), order="F")
    for j, i in enumerate(idx):
        s[i, j] = 1.0
    return s


def random_spd(n, rng):  # tests/helpers.hpp:19-22
    b = rng.gaussian_matrix(n, n)
    return b @ b.T + 0.5 * n * np.eye(n)


def kron(a, b):
    return np.kron(a, b)


def kkt_projection(x, w, c, d):  # tests/helpers.hpp:48-65
    n = x.shape[0]
    nn = n * n
    m = c.shape[0]
    w_inv = np.linalg.inv(w)
    g = kron(w_inv, w_inv)
    kkt = np.zeros((nn + m, nn + m))
    kkt[:nn, :nn] = 2.0 * g
    kkt[:nn, nn:] = c.T
    kkt[nn:, :nn] = c
    rhs = np.zeros(nn + m)
    rhs[nn:] = d
    sol = np.linalg.lstsq(kkt, rhs, rcond=None)[0]
    return x + sol[:nn].reshape((n, n), order="F")


def sym_oracle(x, a, s, w):  # tests/helpers.hpp:87-106
    n = x.shape[0]
    as_ = a @ s
    mc = n * as_.shape[1]
    ms = n * (n - 1) // 2
    c = np.zeros((mc + ms, n * n))
    c[:mc] = kron(as_.T, np.eye(n))
    d = np.zeros(mc + ms)
    d[:mc] = (s - x @ as_).reshape(-1, order="F")
    row = mc
    for i in range(n):
        for j in range(i + 1, n):
            c[row, j * n + i] = 1.0
            c[row, i * n + j] = -1.0
            d[row] = x[j, i] - x[i, j]
            row += 1
    return kkt_projection(x, w, c, d)


# ---------------------------------------------------------------- bfgs_step --
def test_bfgs_hand_fixture():  # test_qn_updates.cpp:199-207
    a = fixture_a()
    stepped = O.bfgs_step(np.eye(2), a, coordinate_sketch(2, [0]))
    expected = np.array([[0.75, -0.5], [-0.5, 1.0]])
    assert np.linalg.norm(stepped - expected) <= 1e-12


def test_bfgs_equals_kkt_oracle():  # test_qn_updates.cpp:209-211
    a = fixture_a()
    x = np.eye(2)
    s = coordinate_sketch(2, [0])
    stepped = O.bfgs_step(x, a, s)
    oracle = sym_oracle(x, a, s, np.linalg.inv(a))
    assert np.linalg.norm(stepped - oracle) <= 1e-8


def test_bfgs_recurrence_and_pd():  # test_qn_updates.cpp:213-228
    rng = O.RngStream(41)
    big = random_spd(5, rng)
    xs = random_spd(5, rng)
    sk = coordinate_sketch(5, [0, 3])
    p = sk @ np.linalg.inv(sk.T @ big @ sk) @ sk.T
    eye = np.eye(5)
    rec = p + (eye - p @ big) @ xs @ (eye - big @ p)
    step5 = O.bfgs_step(xs, big, sk)
    assert np.linalg.norm(step5 - rec) <= 1e-9 * max(1.0, np.linalg.norm(rec))
    assert np.linalg.norm(step5 - step5.T) <= 1e-10
    vals, _ = O.jacobi_eigendecomposition(step5)
    assert vals[0] > 0.0
    assert np.linalg.norm(O.bfgs_step(xs, big, eye) - np.linalg.inv(big)) <= 1e-8


def test_bfgs_full_sketch_one_step():  # acceptance.cpp:51-85 (bfgs leg), n=50, 20 trials
    n = 50
    worst = 0.0
    for trial in range(20):
        rng = O.RngStream(100 + trial)
        _a = rng.gaussian_matrix(n, n)  # general A drawn first (acceptance.cpp:58) keeps the stream aligned
        _w = random_spd(n, rng)
        spd = random_spd(n, rng)
        spd_inv = np.linalg.inv(spd)
        x1 = O.bfgs_step(np.eye(n), spd, np.eye(n))
        worst = max(worst, np.linalg.norm(x1 - spd_inv) / np.linalg.norm(spd_inv))
    assert worst <= 1e-8


def test_bfgs_rank_deficient_gram_raises():  # test_qn_updates.cpp:253-268 (resample contract)
    rng = O.RngStream(47)
    a = random_spd(3, rng)
    with pytest.raises(O.NumericalError):
        O.bfgs_step(np.eye(3), a, np.zeros((3, 1)))
    rep = np.ones((3, 2))
    with pytest.raises(O.NumericalError):
        O.bfgs_step(np.eye(3), a, rep)


def test_run_inverter_bfgs_symmetric():  # test_simi.cpp:163-173
    rng = O.RngStream(67)
    a = random_spd(5, rng)
    res = O.run_inverter_bfgs(a, 2, rule=O.RULE_COORDINATE_BLOCK, tol=0.0, max_iters=30, every_k=10)
    assert np.linalg.norm(res.x - res.x.T) == 0.0
    assert res.max_symmetry_drift < 1e-8
    assert res.termination == 1 and res.k == 30
    # k = 0 baseline then checkpoints at 1, 10, 20, 30 (simi.cpp:361-375)
    assert [h[0] for h in res.history] == [0, 1, 10, 20, 30]
    assert res.history[0][1] == 1.0


def test_run_inverter_checkpoints_and_flops():  # test_simi.cpp:107-121 (checkpoint rule), bfgs flavour
    rng = O.RngStream(3)
    a = random_spd(6, rng)
    res = O.run_inverter_bfgs(a, 2, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=5, every_k=2)
    assert [h[0] for h in res.history] == [0, 1, 2, 4, 5]
    fl = [h[2] for h in res.history]
    assert all(fl[i] > fl[i - 1] for i in range(1, len(fl)))
    assert fl[-1] == pytest.approx(5 * O.flops_bfgs(6, 2))


def test_run_inverter_converges_gaussian():
    rng = O.RngStream(5)
    a = random_spd(12, rng)
    res = O.run_inverter_bfgs(a, 3, rule=O.RULE_GAUSSIAN, tol=1e-8, max_iters=2000, every_k=5, seed=9)
    assert res.termination == 0
    assert np.linalg.norm(a @ res.x - np.eye(12)) <= 1e-6


# ---------------------------------------------------------------- adarbfgs ---
def test_adarbfgs_scalar_fixture():  # test_adarbfgs.cpp:15-23
    nxt = O.adarbfgs_update_factor([[1.0]], [[4.0]], [[1.0]])
    assert nxt[0, 0] == pytest.approx(0.5, rel=1e-12)
    assert (nxt @ nxt.T)[0, 0] == pytest.approx(0.25, rel=1e-12)


def test_adarbfgs_factored_equals_direct():  # test_adarbfgs.cpp:25-35
    rng = O.RngStream(73)
    a = random_spd(6, rng)
    l = np.eye(6) + 0.1 * rng.gaussian_matrix(6, 6)
    x = l @ l.T
    st = rng.gaussian_matrix(6, 2)
    nl = O.adarbfgs_update_factor(l, a, st)
    direct = O.bfgs_step(x, a, l @ st)
    assert np.linalg.norm(nl @ nl.T - direct) <= 1e-8 * max(1.0, np.linalg.norm(direct))


def test_adaptive_block_probabilities_direct():  # test_adarbfgs.cpp:37-52
    rng = O.RngStream(79)
    a = random_spd(6, rng)
    l = np.eye(6) + 0.2 * rng.gaussian_matrix(6, 6)
    p = O.adaptive_block_probabilities(l, a, 2)
    total = np.trace(a @ l @ l.T)
    for i in range(3):
        tr = sum(l[:, j] @ (a @ l[:, j]) for j in (2 * i, 2 * i + 1))
        assert p[i] == pytest.approx(tr / total, rel=1e-10)
    assert abs(p.sum() - 1.0) <= 1e-12


def test_adarbfgs_degenerate_sketch_raises():  # test_adarbfgs.cpp:73-78
    with pytest.raises(O.NumericalError):
        O.adarbfgs_update_factor(np.eye(2), fixture_a(), np.zeros((2, 1)))


def test_adarbfgs_1000_cols_steps_factored_vs_direct():  # acceptance.cpp:306-341
    n = 10
    rng = O.RngStream(700)
    a = random_spd(n, rng)
    l = np.eye(n)
    worst, min_lambda = 0.0, np.inf
    for _ in range(1000):
        p = O.adaptive_block_probabilities(l, a, 2)
        b = rng.categorical(p)
        st = coordinate_sketch(n, [2 * b, 2 * b + 1])
        try:
            nl = O.adarbfgs_update_factor(l, a, st)
        except O.NumericalError:
            continue
        direct = O.bfgs_step(l @ l.T, a, l @ st)
        xn = nl @ nl.T
        worst = max(worst, np.linalg.norm(xn - direct) / max(1.0, np.linalg.norm(direct)))
        min_lambda = min(min_lambda, np.linalg.eigvalsh(xn).min())
        l = nl
    assert min_lambda > 0.0 and worst <= 1e-8


@pytest.mark.parametrize("rule", [O.ADA_COLS, O.ADA_GAUSS, O.ADA_COLS_UNIFORM])
def test_run_adarbfgs_converges(rule):  # test_adarbfgs.cpp:94-112
    rng = O.RngStream(89)
    a = random_spd(10, rng)
    res = O.run_adarbfgs(a, 2, rule=rule, tol=1e-6, max_iters=4000, every_k=20, seed=5)
    assert res.termination == 0
    x = res.x @ res.x.T
    assert np.linalg.norm(a @ x - np.eye(10)) <= 1e-5 * np.linalg.norm(a) * 10
    assert np.linalg.eigvalsh(x).min() > 0.0
    assert res.history[0][1] == 1.0


def test_run_adarbfgs_config_validation():  # test_adarbfgs.cpp:114-133
    with pytest.raises(O.ConfigError):
        O.run_adarbfgs(fixture_a(), 1, rule=O.ADA_GAUSS, tol=-1.0)
    with pytest.raises(O.ConfigError):
        O.run_adarbfgs(fixture_a(), 3, rule=O.ADA_GAUSS)


# ---------------------------------------------------------------- linalg -----
def test_jacobi_recovers_spectrum():  # test_linalg.cpp:14-28
    rng = O.RngStream(11)
    b = rng.gaussian_matrix(6, 6)
    m = 0.5 * (b + b.T)
    vals, vecs = O.jacobi_eigendecomposition(m)
    assert np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - m) <= 1e-10 * max(1.0, np.linalg.norm(m))
    assert np.linalg.norm(vecs.T @ vecs - np.eye(6)) <= 1e-12
    assert np.all(np.diff(vals) >= 0)
    vals, _ = O.jacobi_eigendecomposition(np.diag([3.0, 1.0, 2.0]))
    assert vals[0] == pytest.approx(1.0, rel=1e-14) and vals[2] == pytest.approx(3.0, rel=1e-14)


def test_sym_inv_sqrt_identity_and_floor():  # test_linalg.cpp:85-101
    rng = O.RngStream(5)
    m = random_spd(5, rng)
    ir = O.sym_inv_sqrt(m)
    assert np.linalg.norm(ir @ m @ ir - np.eye(5)) <= 1e-9
    singular = np.zeros((2, 2))
    singular[0, 0] = 1.0
    with pytest.raises(O.NumericalError):
        O.sym_inv_sqrt(singular)


# ---------------------------------------------------------------- rng --------
def test_rng_determinism_and_substreams():  # test_sketching_rates.cpp:240-257
    a = O.RngStream(7).gaussian_matrix(8, 3)
    b = O.RngStream(7).gaussian_matrix(8, 3)
    assert np.array_equal(a, b)
    s1 = O.RngStream(7).substream(2).uniform_matrix(4, 4)
    s2 = O.RngStream(7).substream(2).uniform_matrix(4, 4)
    assert np.array_equal(s1, s2)
    assert not np.array_equal(s1, O.RngStream(7).substream(3).uniform_matrix(4, 4))


def test_rng_categorical_frequencies():  # test_sketching_rates.cpp:226-238 (4 sigma)
    rng = O.RngStream(13)
    p = np.array([0.1, 0.2, 0.3, 0.4])
    draws = 20000
    counts = np.zeros(4)
    for _ in range(draws):
        counts[rng.categorical(p)] += 1
    sigma = np.sqrt(draws * p * (1 - p))
    assert np.all(np.abs(counts - draws * p) <= 4 * sigma)


def test_uniform_subset_distinct():
    rng = O.RngStream(21)
    for _ in range(50):
        idx = rng.uniform_subset(64, 16)
        assert len(set(idx.tolist())) == 16 and idx.min() >= 0 and idx.max() < 64


# ------------------------------------------------- row f3: psb / aip / dfp --
def random_symmetric(n, rng):  # tests/helpers.hpp:24-27
    b = rng.gaussian_matrix(n, n)
    return 0.5 * (b + b.T)


def row_oracle(x, a, s, w):  # tests/helpers.hpp:69-75
    n = x.shape[0]
    sa = s.T @ a
    return kkt_projection(x, w, kron(np.eye(n), sa), (s.T - sa @ x).reshape(-1, order="F"))


def test_psb_matches_symmetric_oracle():  # test_qn_updates.cpp:119-132
    rng = O.RngStream(23)
    a = random_symmetric(4, rng)
    x = random_symmetric(4, rng)
    s = coordinate_sketch(4, [1, 2])
    stepped = O.psb_step(x, a, s)
    oracle = sym_oracle(x, a, s, np.eye(4))
    assert np.linalg.norm(stepped - oracle) <= 1e-8 * max(1.0, np.linalg.norm(oracle))
    assert np.linalg.norm(stepped - stepped.T) <= 1e-10
    assert np.linalg.norm(stepped @ a @ s - s) <= 1e-9


def test_aip_equals_row_update_with_inverse_weight():  # test_qn_updates.cpp:160-174
    rng = O.RngStream(31)
    a = random_spd(4, rng)
    x = random_symmetric(4, rng)
    s = coordinate_sketch(4, [0, 3])
    stepped = O.aip_step(x, a, s)
    a_inv = O.lu_inverse(a)
    oracle = row_oracle(x, a, s, a_inv)
    assert np.linalg.norm(stepped - oracle) <= 1e-7 * max(1.0, np.linalg.norm(oracle))
    assert np.linalg.norm(s.T @ a @ stepped - s.T) <= 1e-9


def test_dfp_full_sketch_recurrence_and_woodbury_pair():  # test_qn_updates.cpp:176-197
    rng = O.RngStream(37)
    a = random_spd(4, rng)
    x, x_inv = np.eye(4), np.eye(4)
    full_p, full_i = O.dfp_step(x, x_inv, a, np.eye(4))
    assert np.linalg.norm(full_p - a) <= 1e-9 * np.linalg.norm(a)
    assert np.linalg.norm(full_i @ a - np.eye(4)) <= 1e-8
    s = coordinate_sketch(4, [1, 2])
    nxt_p, nxt_i = O.dfp_step(x, x_inv, a, s)
    omega = s @ O.lu_inverse(s.T @ a @ s) @ s.T
    eye = np.eye(4)
    expected = a + (eye - a @ omega) @ (x - a) @ (eye - omega @ a)
    assert np.linalg.norm(nxt_p - expected) <= 1e-9 * max(1.0, np.linalg.norm(expected))
    assert np.linalg.norm(nxt_p - nxt_p.T) <= 1e-10
    assert np.linalg.norm(nxt_i - O.lu_inverse(nxt_p)) <= 1e-8


def test_rank_deficient_grams_raise_for_psb():  # test_qn_updates.cpp:253-261
    rng = O.RngStream(47)
    a = rng.gaussian_matrix(3, 3)
    with pytest.raises(O.NumericalError):
        O.psb_step(np.eye(3), a, np.zeros((3, 1)))
    with pytest.raises(O.NumericalError):
        O.aip_step(np.eye(3), random_spd(3, rng), np.ones((3, 2)))


def test_lu_inverse_general():
    rng = O.RngStream(5)
    m = rng.gaussian_matrix(7, 7) + 3 * np.eye(7)
    assert np.allclose(O.lu_inverse(m) @ m, np.eye(7), atol=1e-12)


@pytest.mark.parametrize("update", [O.UPDATE_PSB, O.UPDATE_AIP, O.UPDATE_DFP, O.UPDATE_BFGS])
def test_run_inverter_named_updates_converge(update):  # test_simi.cpp convergence contract, per update
    rng = O.RngStream(53)
    a = random_spd(12, rng)
    res, xi = O.run_inverter(a, 3, update=update, rule=O.RULE_COORDINATE_BLOCK, tol=1e-8, max_iters=4000,
                             every_k=10, seed=2)
    assert res.termination == 0
    tracked = xi if update == O.UPDATE_DFP else res.x
    assert np.linalg.norm(np.eye(12) - a @ tracked) <= 1e-7 * np.linalg.norm(np.eye(12) - a)
    assert res.history[0][1] == 1.0
    if update != O.UPDATE_AIP:
        assert np.array_equal(res.x, res.x.T)


def test_run_inverter_bfgs_general_equals_bfgs_driver():
    rng = O.RngStream(59)
    a = random_spd(16, rng)
    r1, _ = O.run_inverter(a, 4, update=O.UPDATE_BFGS, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=25, every_k=5, seed=9)
    r2 = O.run_inverter_bfgs(a, 4, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=25, every_k=5, seed=9)
    assert np.array_equal(r1.x, r2.x)
    assert r1.history == [(k, r, f, r1.history[i][3]) for i, (k, r, f, _) in enumerate(r2.history)]


def test_flop_polynomials():  # flops.cpp:22-46
    assert O.flops_named(O.UPDATE_PSB, 3, 2) == 8 * 18 + 8 * 12 + 16 + 6 + 27
    assert O.flops_named(O.UPDATE_AIP, 3, 2) == 6 * 18 + 4 * 12 + 16 + 6 + 9
    assert O.flops_named(O.UPDATE_DFP, 3, 2) == 14 * 18 + 14 * 12 + 32 + 54


# ---------------------------------------------------- row f4: baselines --
def test_newton_schulz_scalar_and_quadratic_identity():  # test_baselines.cpp:14-33
    a = np.array([[2.0]])
    x = O.newton_schulz_step(np.array([[0.4]]), a)
    assert x[0, 0] == pytest.approx(0.48, rel=1e-14)
    x = O.newton_schulz_step(x, a)
    assert x[0, 0] == pytest.approx(0.4992, rel=1e-14)
    assert O.newton_schulz_init(a)[0, 0] == pytest.approx(0.495, rel=1e-8)
    rng = O.RngStream(91)
    m = random_spd(6, rng)
    x0 = O.newton_schulz_init(m, 3)
    res = np.eye(6) - m @ x0
    x1 = O.newton_schulz_step(x0, m)
    assert np.linalg.norm(np.eye(6) - m @ x1 - res @ res) <= 1e-10 * max(1.0, np.linalg.norm(res))


def test_minimal_residual_scalar_and_init():  # test_baselines.cpp:35-50
    a = np.array([[2.0]])
    xo, _, alpha, stg = O.mr_step_cached(np.array([[0.25]]), np.eye(1) - 0.25 * a, a)
    assert xo[0, 0] == pytest.approx(0.5, rel=1e-14) and alpha == pytest.approx(2.0) and not stg
    init = O.mr_init(np.diag([1.0, 3.0]))
    assert np.linalg.norm(init - 0.4 * np.eye(2)) <= 1e-14
    with pytest.raises(O.ConfigError):
        O.mr_init(np.zeros((2, 2)))


def test_minimal_residual_monotone():  # test_baselines.cpp:52-71
    rng = O.RngStream(93)
    a = random_spd(8, rng)
    x = O.mr_init(a)
    r = np.eye(8) - a @ x
    prev = np.linalg.norm(r)
    for _ in range(1000):
        xn, rn, _, stg = O.mr_step_cached(x, r, a)
        if stg:
            break
        x, r = xn, rn
        cur = np.linalg.norm(r)
        assert cur <= prev * (1.0 + 1e-12)
        prev = cur
    assert np.linalg.norm(r - (np.eye(8) - a @ x)) <= 1e-8 * max(1.0, prev)
    assert prev <= 0.5 * np.linalg.norm(np.eye(8) - a @ O.mr_init(a))


def test_mr_stagnates_at_exact_inverse():  # test_baselines.cpp:73-83
    d = np.diag([2.0, 4.0])
    xo, _, alpha, stg = O.mr_step_cached(np.diag([0.5, 0.25]), np.zeros((2, 2)), d)
    assert stg and alpha == 0.0 and np.array_equal(xo, np.diag([0.5, 0.25]))


def test_run_baseline_converges_and_contract():  # test_baselines.cpp:85-123, 125-146
    rng = O.RngStream(97)
    a = random_spd(12, rng)
    ns = O.run_baseline(a, method=O.BASELINE_NS, tol=1e-8, max_iters=200, every_k=5)
    assert ns.termination == 0
    assert np.linalg.norm(a @ ns.x - np.eye(12)) <= 1e-6 * np.linalg.norm(a)
    assert ns.history[0][1] == 1.0 and ns.history[-1][2] > 0.0
    mr = O.run_baseline(a, method=O.BASELINE_MR, tol=1e-2, max_iters=5000, every_k=25)
    assert mr.termination == 0 and mr.history[-1][1] <= 1e-2
    stiff = random_spd(10, O.RngStream(101))
    div = O.run_baseline(stiff, method=O.BASELINE_NS, max_iters=200, x0=np.eye(10))
    assert div.termination == 2 and "diverged" in O.lib().or_last_error().decode()
    with pytest.raises(O.ConfigError):
        O.run_baseline(a, tol=-1.0)
    exact = O.run_baseline(np.diag([2.0, 4.0]), x0=np.diag([0.5, 0.25]))
    assert exact.termination == 0 and exact.history[0][1] == 0.0


def test_spectral_norm_estimate():
    rng = O.RngStream(3)
    m = rng.gaussian_matrix(9, 6)
    est = O.spectral_norm_estimate(m, 100, 1)
    assert est <= np.linalg.norm(m, 2) * (1 + 1e-12)
    assert est == pytest.approx(np.linalg.norm(m, 2), rel=1e-6)
