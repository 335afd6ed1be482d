"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same A, seed and sketches.  Bars (north_star): coordinate indices bit-exact,
FP64 iterate relative Frobenius ≤ 1e-9 after 50 iterations, residual trace
within 1% relative.  Reference KATs are re-run on the GPU path.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-9  # relative Frobenius on the iterate (north_star)
TRACE_TOL = 0.01  # residual trace, relative (north_star)


@pytest.fixture(scope="module")
def si():
    import paper_1602_01768_b200 as si

    return si


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def trace_gap(got, ref, floor=1e-10):
    """Max relative gap of two residual traces over the points above the rounding
    floor; below it (finite termination at machine precision) both must be tiny."""
    got, ref = np.asarray(got), np.asarray(ref)
    live = ref > floor
    assert np.all(got[~live] <= 1e3 * floor)
    return float(np.max(np.abs(got[live] - ref[live]) / ref[live])) if live.any() else 0.0


def random_spd(n, rng):  # tests/helpers.hpp:19-22
    b = rng.gaussian_matrix(n, n)
    return b @ b.T + 0.5 * n * np.eye(n)


def coordinate_sketch(n, idx):
    s = np.zeros((n, len(idx)), order="F")
    for j, i in enumerate(idx):
        s[i, j] = 1.0
    return s


# ------------------------------------------------------------ step kernels --
def test_bfgs_hand_fixture_gpu(si):  # test_qn_updates.cpp:199-207
    a = np.array([[2.0, 1.0], [1.0, 2.0]])
    out = si.bfgs_step(np.eye(2), a, coordinate_sketch(2, [0]))
    assert np.linalg.norm(out - np.array([[0.75, -0.5], [-0.5, 1.0]])) <= 1e-12


def test_bfgs_recurrence_and_full_sketch_gpu(si):  # test_qn_updates.cpp:213-228
    rng = O.RngStream(41)
    big = random_spd(5, rng)
    xs = random_spd(5, rng)
    sk = coordinate_sketch(5, [0, 3])
    p = sk @ np.linalg.inv(sk.T @ big @ sk) @ sk.T
    eye = np.eye(5)
    rec = p + (eye - p @ big) @ xs @ (eye - big @ p)
    step5 = si.bfgs_step(xs, big, sk)
    assert np.linalg.norm(step5 - rec) <= 1e-9 * max(1.0, np.linalg.norm(rec))
    assert np.linalg.norm(step5 - step5.T) <= 1e-10
    assert np.linalg.eigvalsh(step5).min() > 0
    assert np.linalg.norm(si.bfgs_step(xs, big, eye) - np.linalg.inv(big)) <= 1e-8


@pytest.mark.parametrize("n,q", [(1, 1), (7, 3), (37, 5), (130, 17), (256, 32), (300, 64), (513, 128), (640, 130),
                                 (700, 300), (1100, 520)])
def test_bfgs_step_matches_oracle(si, n, q):
    rng = O.RngStream(1000 + n + q)
    a = random_spd(n, rng)
    x = random_spd(n, rng) / n
    s = rng.gaussian_matrix(n, q)
    ref = O.bfgs_step(x, a, s)
    got = si.bfgs_step(x, a, s)
    assert rel(got, ref) <= 1e-11
    assert np.array_equal(got, got.T)  # written exactly symmetric
    # sketch-and-project consistency: X⁺ A S = S
    assert np.linalg.norm(got @ (a @ s) - s) <= 1e-9 * max(1.0, np.linalg.norm(s))


def test_bfgs_resample_signal(si):  # test_qn_updates.cpp:253-268
    rng = O.RngStream(47)
    a = random_spd(3, rng)
    with pytest.raises(si.GramRankDeficientError):
        si.bfgs_step(np.eye(3), a, np.zeros((3, 1)))
    with pytest.raises(si.GramRankDeficientError):
        si.bfgs_step(np.eye(3), a, np.ones((3, 2)))


def test_bfgs_full_sketch_one_step_gpu(si):  # acceptance.cpp:51-85 (bfgs leg)
    n = 50
    worst = 0.0
    for trial in range(5):
        rng = O.RngStream(100 + trial)
        rng.gaussian_matrix(n, n)
        random_spd(n, rng)
        spd = random_spd(n, rng)
        inv = np.linalg.inv(spd)
        worst = max(worst, rel(si.bfgs_step(np.eye(n), spd, np.eye(n)), inv))
    assert worst <= 1e-8


def test_adarbfgs_scalar_fixture_gpu(si):  # test_adarbfgs.cpp:15-23
    nxt = si.adarbfgs_update_factor([[1.0]], [[4.0]], [[1.0]])
    assert nxt[0, 0] == pytest.approx(0.5, rel=1e-12)


@pytest.mark.parametrize("n,q,gauss", [(6, 2, True), (40, 5, True), (128, 16, False), (200, 64, False),
                                       (300, 96, False), (320, 128, False), (400, 160, True), (600, 256, False)])
def test_adarbfgs_update_matches_oracle(si, n, q, gauss):  # test_adarbfgs.cpp:25-35 + oracle
    rng = O.RngStream(73 + n)
    a = random_spd(n, rng)
    l = np.eye(n) + 0.1 * rng.gaussian_matrix(n, n) / np.sqrt(n)
    if gauss:
        st = rng.gaussian_matrix(n, q)
    else:
        st = coordinate_sketch(n, list(rng.uniform_subset(n, q)))
    ref = O.adarbfgs_update_factor(l, a, st)
    got = si.adarbfgs_update_factor(l, a, st)
    assert rel(got, ref) <= 1e-10
    direct = O.bfgs_step(l @ l.T, a, l @ st)
    assert np.linalg.norm(got @ got.T - direct) <= 1e-8 * max(1.0, np.linalg.norm(direct))


def test_adarbfgs_degenerate_raises(si):  # test_adarbfgs.cpp:73-78
    with pytest.raises(si.NumericalError):
        si.adarbfgs_update_factor(np.eye(2), [[2.0, 1.0], [1.0, 2.0]], np.zeros((2, 1)))


def test_adaptive_block_probabilities_gpu(si):  # test_adarbfgs.cpp:37-52
    rng = O.RngStream(79)
    a = random_spd(64, rng)
    l = np.eye(64) + 0.2 * rng.gaussian_matrix(64, 64) / 8
    blocks = si.contiguous_partition(64, 8)
    got = si.adaptive_block_probabilities(l, a, blocks)
    ref = O.adaptive_block_probabilities(l, a, 8)
    assert np.allclose(got, ref, rtol=1e-12, atol=0)
    assert abs(got.sum() - 1.0) <= 1e-12


# ------------------------------------------------------------------ drivers --
def test_run_inverter_config1_parity(si):
    """BASELINE config 1 (n=1024, q=32, Gaussian, seed 0), 50 iterations, residual every iteration."""
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(1024, seed=0)
    iters = 50
    ref = O.run_inverter_bfgs(a, 32, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=iters, every_k=1, seed=0)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    cfg = si.InverterConfig(prob, si.SketchRule.gaussian(32), tol=0.0, max_iters=iters, seed=0,
                            track=si.TrackOptions(residual_every_k=1))
    res = si.run_inverter(cfg)
    assert res.termination == si.Termination.max_iters and res.state.k == iters
    assert rel(res.state.x, ref.x) <= ITER_TOL
    got_tr = np.array([h.residual for h in res.state.history])
    ref_tr = np.array([h[1] for h in ref.history])
    assert [h.k for h in res.state.history] == [h[0] for h in ref.history]
    assert trace_gap(got_tr, ref_tr) <= TRACE_TOL
    assert trace_gap(got_tr, ref_tr) <= 1e-9  # far inside the bar
    flops = [h.flops for h in res.state.history]
    assert flops[-1] == pytest.approx(iters * si.flops_bfgs(1024, 32))


def test_run_inverter_coordinate_block_indices(si):
    rng = O.RngStream(67)
    a = random_spd(40, rng)
    ref = O.run_inverter_bfgs(a, 4, rule=O.RULE_COORDINATE_BLOCK, tol=0.0, max_iters=60, every_k=5, seed=3)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    res = si.run_inverter(si.InverterConfig(prob, si.SketchRule.coordinate_block(40, 4), tol=0.0, max_iters=60,
                                            seed=3, track=si.TrackOptions(residual_every_k=5)))
    assert rel(res.state.x, ref.x) <= ITER_TOL
    assert np.array_equal(res.state.x, res.state.x.T)
    assert res.state.max_symmetry_drift < 1e-8


def test_run_inverter_converges_and_validates(si):
    rng = O.RngStream(5)
    a = random_spd(48, rng)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    res = si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(6), tol=1e-8, max_iters=3000, seed=9,
                                            track=si.TrackOptions(residual_every_k=5)))
    assert res.termination == si.Termination.tol_reached
    assert np.linalg.norm(a @ res.state.x - np.eye(48)) <= 1e-6 * np.linalg.norm(a)
    with pytest.raises(si.ConfigError):
        si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(60)))
    with pytest.raises(si.ConfigError):
        si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(2), tol=-1.0))
    with pytest.raises(si.ConfigError):
        si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.general), si.SketchRule.gaussian(2)))
    xs = np.eye(48)
    xs[0, 1] = 1.0
    with pytest.raises(si.ConfigError):
        si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(2), x0=xs))


def test_run_inverter_full_sketch_terminates(si):  # test_simi.cpp:94-105 flavour
    rng = O.RngStream(8)
    a = random_spd(16, rng)
    res = si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.spd),
                                            si.SketchRule.coordinate_block(16, 16), tol=1e-10))
    assert res.termination == si.Termination.tol_reached and res.state.k == 1
    assert np.linalg.norm(res.state.x - np.linalg.inv(a)) <= 1e-10 * np.linalg.norm(np.linalg.inv(a))


def test_run_inverter_checkpoint_callback(si):
    rng = O.RngStream(3)
    a = random_spd(32, rng)
    seen = []
    res = si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.gaussian(4),
                                            tol=0.0, max_iters=7, track=si.TrackOptions(residual_every_k=3),
                                            on_checkpoint=seen.append))
    assert [p.k for p in seen] == [0, 1, 3, 6, 7] == [h.k for h in res.state.history]


@pytest.mark.parametrize("rule", ["cols", "uniform", "gauss"])
def test_run_adarbfgs_parity(si, rule):
    rng = O.RngStream(89)
    n, q = 96, 8
    a = random_spd(n, rng)
    orule = {"cols": O.ADA_COLS, "uniform": O.ADA_COLS_UNIFORM, "gauss": O.ADA_GAUSS}[rule]
    srule = {"cols": si.SketchRule.adaptive_cols(n, q), "uniform": si.SketchRule.adaptive_cols_uniform(q),
             "gauss": si.SketchRule.adaptive_gauss(q)}[rule]
    iters = 50
    ref = O.run_adarbfgs(a, q, rule=orule, tol=0.0, max_iters=iters, every_k=5, seed=5)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), srule, tol=0.0, max_iters=iters, seed=5,
                                       track=si.TrackOptions(residual_every_k=5)))
    assert res.state.k == iters
    assert rel(res.state.l, ref.x) <= ITER_TOL
    got_tr = np.array([h.residual for h in res.state.history])
    ref_tr = np.array([h[1] for h in ref.history])
    assert trace_gap(got_tr, ref_tr) <= TRACE_TOL
    assert rel(res.state.x, res.state.l @ res.state.l.T) <= 1e-13


@pytest.mark.parametrize("refresh", ["1", "7", "100000"])
def test_eq82_incremental_diagonal_parity(si, refresh, monkeypatch):
    """Eq. 8.2 probabilities from the carried diag(LᵀAL) (App. C3) draw the same
    blocks as the reference's exact A·L every iteration: 150 iterations over a
    ragged partition (n = 100, q = 8: last block 4 wide), same iterate."""
    monkeypatch.setenv("SI_PDIAG_REFRESH", refresh)
    rng = O.RngStream(23)
    n, q, iters = 100, 8, 150
    a = random_spd(n, rng)
    ref = O.run_adarbfgs(a, q, rule=O.ADA_COLS, tol=0.0, max_iters=iters, every_k=10, seed=2)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.adaptive_cols(n, q),
                                       tol=0.0, max_iters=iters, seed=2, track=si.TrackOptions(residual_every_k=10)))
    assert res.state.k == iters
    assert rel(res.state.l, ref.x) <= ITER_TOL
    assert trace_gap([h.residual for h in res.state.history], [h[1] for h in ref.history]) <= TRACE_TOL


def test_eq82_incremental_diagonal_from_x0(si, monkeypatch):
    monkeypatch.setenv("SI_PDIAG_REFRESH", "1000")
    rng = O.RngStream(29)
    n, q, iters = 64, 8, 60
    a = random_spd(n, rng)
    l0 = np.eye(n) + 0.01 * rng.gaussian_matrix(n, n)
    ref = O.run_adarbfgs(a, q, rule=O.ADA_COLS, tol=0.0, max_iters=iters, every_k=10, seed=4, l0=l0)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.adaptive_cols(n, q),
                                       tol=0.0, max_iters=iters, seed=4, l0=l0,
                                       track=si.TrackOptions(residual_every_k=10)))
    assert rel(res.state.l, ref.x) <= ITER_TOL


def test_run_adarbfgs_converges(si):  # test_adarbfgs.cpp:94-112
    rng = O.RngStream(89)
    a = random_spd(10, rng)
    for rule in (si.SketchRule.adaptive_cols(10, 2), si.SketchRule.adaptive_gauss(2)):
        res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), rule, tol=1e-6, max_iters=4000,
                                           seed=5, track=si.TrackOptions(residual_every_k=20)))
        assert res.termination == si.Termination.tol_reached
        assert np.linalg.eigvalsh(res.state.x).min() > 0
        assert res.state.history[0].residual == 1.0


# -------------------------------------------------------- device RNG mode --
def test_device_sketch_statistics_and_convergence(si):
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(256, seed=1)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    res = si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian_device(16), tol=0.0, max_iters=200, seed=11,
                                            track=si.TrackOptions(residual_every_k=50)))
    ref = O.run_inverter_bfgs(a, 16, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=200, every_k=50, seed=11)
    # different random stream: compare convergence statistically (within 25% after 200 its)
    g, r = res.state.history[-1].residual, ref.history[-1][1]
    assert 0.75 * r <= g <= 1.33 * r
    assert np.array_equal(res.state.x, res.state.x.T)


@pytest.mark.parametrize("n,q,every,iters", [(200, 12, 1, 12), (200, 12, 7, 30), (200, 12, 10, 10), (200, 12, 4, 9),
                                             (301, 100, 3, 7), (333, 130, 5, 11)])
def test_batched_device_run_matches_eager_loop(si, n, q, every, iters, monkeypatch):
    """run_inverter with device sketches enqueues the iterations between checkpoints
    back to back (advance_batch_kernel keeps the accounting on the device); the eager
    per-iteration loop (SI_RUN_EAGER=1) must give the same k, history and iterate
    (odd n, a padded K-FACTOR block at q = 100, the GEMM-recursion inverse at q = 130)."""
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(n, seed=3)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)

    def run():
        return si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian_device(q), tol=0.0, max_iters=iters,
                                                 seed=4, track=si.TrackOptions(residual_every_k=every)))

    batched = run()
    monkeypatch.setenv("SI_RUN_EAGER", "1")
    eager = run()
    assert batched.state.k == eager.state.k == iters
    assert [h.k for h in batched.state.history] == [h.k for h in eager.state.history]
    assert [h.residual for h in batched.state.history] == [h.residual for h in eager.state.history]
    assert [h.flops for h in batched.state.history] == [h.flops for h in eager.state.history]
    assert np.array_equal(batched.state.x, eager.state.x)


def test_batched_device_run_tolerance_and_rejections(si, monkeypatch):
    """Tolerance stop at a checkpoint, and the redraw contract on a numerically
    rank-one problem — batched and eager agree on
    the termination, k, the redraw count and the message."""
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(128, seed=5)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    outs = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("SI_RUN_EAGER", "1")
        outs.append(si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian_device(16), tol=0.3,
                                                      max_iters=5000, seed=6,
                                                      track=si.TrackOptions(residual_every_k=5))))
    assert outs[0].termination == outs[1].termination == si.Termination.tol_reached
    assert outs[0].state.k == outs[1].state.k and outs[0].state.k % 5 == 0
    assert np.array_equal(outs[0].state.x, outs[1].state.x)
    monkeypatch.delenv("SI_RUN_EAGER")
    # numerically rank-one Gram matrices: most sketched Grams fail the PD test (the
    # Schur pivots after the first are rounding noise), so draws are rejected and
    # redrawn; both loops must meet the same pivots and reach the same outcome
    lp = si.ProblemMatrix(np.diag(np.r_[1.0, np.full(39, 1e-300)]), si.Symmetry.spd)
    res = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("SI_RUN_EAGER", "1")
        res.append(si.run_inverter(si.InverterConfig(lp, si.SketchRule.gaussian_device(4), tol=0.0, max_iters=10,
                                                     seed=1, max_redraws=3)))
    assert res[0].termination == res[1].termination
    assert res[0].state.k == res[1].state.k
    assert res[0].message == res[1].message
    assert res[0].state.redraws == res[1].state.redraws > 0
    assert [h.residual for h in res[0].state.history] == [h.residual for h in res[1].state.history]


@pytest.mark.parametrize("rule,every,iters", [("uniform", 10, 35), ("uniform", 1, 6), ("gauss_device", 7, 20)])
def test_batched_adarbfgs_matches_eager_loop(si, rule, every, iters, monkeypatch):
    """run_adarbfgs enqueues up to 64 attempts between checkpoints (host-drawn uniform
    index sets uploaded once; device Philox S̃) — same k, history and factor as the
    per-iteration loop (SI_RUN_EAGER=1)."""
    rng = O.RngStream(41)
    n, q = 72, 6
    a = random_spd(n, rng)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    srule = si.SketchRule.adaptive_cols_uniform(q) if rule == "uniform" else si.SketchRule.adaptive_gauss_device(q)

    def run():
        return si.run_adarbfgs(si.AdaConfig(prob, srule, tol=0.0, max_iters=iters, seed=3,
                                            track=si.TrackOptions(residual_every_k=every)))

    batched = run()
    monkeypatch.setenv("SI_RUN_EAGER", "1")
    eager = run()
    assert batched.state.k == eager.state.k == iters
    assert [h.k for h in batched.state.history] == [h.k for h in eager.state.history]
    assert [h.residual for h in batched.state.history] == [h.residual for h in eager.state.history]
    assert np.array_equal(batched.state.l, eager.state.l)


def test_batched_adarbfgs_rejections_match_eager(si, monkeypatch):
    """A = diag(1, …, 1, 1e-300): every coordinate Gram containing the last index is
    numerically singular and its inverse square root is rejected (the resample signal),
    the others are accepted — batched and eager loops meet the same draws, redraws and
    iterates."""
    n, q = 40, 4
    prob = si.ProblemMatrix(np.diag(np.r_[np.ones(n - 1), 1e-300]), si.Symmetry.spd)
    outs = []
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("SI_RUN_EAGER", "1")
        outs.append(si.run_adarbfgs(si.AdaConfig(prob, si.SketchRule.adaptive_cols_uniform(q), tol=0.0, max_iters=30,
                                                 seed=8, max_redraws=100, track=si.TrackOptions(residual_every_k=10))))
    assert outs[0].termination == outs[1].termination
    assert outs[0].state.k == outs[1].state.k
    assert outs[0].state.redraws == outs[1].state.redraws > 0
    assert [h.residual for h in outs[0].state.history] == [h.residual for h in outs[1].state.history]
    assert np.array_equal(outs[0].state.l, outs[1].state.l, equal_nan=True)


def test_workspace_reuse_and_release(si):
    """run_inverter / run_adarbfgs keep their workspace in the context: a rerun of the same
    shape gives the same result, and releasing the cache changes nothing but memory."""
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(160, seed=4)
    ctx = si.Context(0)
    prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
    cfg = si.InverterConfig(prob, si.SketchRule.gaussian_device(8), tol=0.0, max_iters=9, seed=2,
                            track=si.TrackOptions(residual_every_k=4))
    r1 = si.run_inverter(cfg)
    r2 = si.run_inverter(cfg)
    ctx.release_workspaces()
    r3 = si.run_inverter(cfg)
    assert np.array_equal(r1.state.x, r2.state.x) and np.array_equal(r1.state.x, r3.state.x)
    acfg = si.AdaConfig(prob, si.SketchRule.adaptive_cols_uniform(8), tol=0.0, max_iters=7, seed=3,
                        track=si.TrackOptions(residual_every_k=3))
    l1 = si.run_adarbfgs(acfg).state.l
    l2 = si.run_adarbfgs(acfg).state.l
    ctx.release_workspaces()
    l3 = si.run_adarbfgs(acfg).state.l
    assert np.array_equal(l1, l2) and np.array_equal(l1, l3)


def test_solver_step_matches_driver(si):
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(192, seed=2)
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    sol = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian(8), seed=4)
    for _ in range(10):
        sol.step(1)
    ref = O.run_inverter_bfgs(a, 8, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=10, every_k=10, seed=4)
    assert rel(sol.iterate(), ref.x) <= ITER_TOL
    assert sol.residual() == pytest.approx(O.residual(a, ref.x), rel=1e-9)


# ------------------------------------------------------------- sparse (CSR) --
@pytest.mark.parametrize("cfg", ["laplacian", "banded"])
def test_csr_problem_matches_dense(si, cfg):
    from paper_1602_01768_b200 import generators as G

    if cfg == "laplacian":
        n = 144
        rp, ci, v = G.config4_csr(n)
    else:
        n = 300
        rp, ci, v = G.config5_csr(n, half_bandwidth=16)
    dense = G.csr_to_dense(n, rp, ci, v)
    prob = si.ProblemMatrix(csr=(rp, ci, v), n=n, symmetry=si.Symmetry.spd)
    assert np.array_equal(prob.data(), dense)
    res = si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(12), tol=0.0, max_iters=50, seed=0,
                                            track=si.TrackOptions(residual_every_k=10)))
    ref = O.run_inverter_bfgs(dense, 12, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=50, every_k=10, seed=0)
    assert rel(res.state.x, ref.x) <= ITER_TOL
    tr = np.array([h.residual for h in res.state.history])
    rtr = np.array([h[1] for h in ref.history])
    assert trace_gap(tr, rtr) <= TRACE_TOL
    # AdaRBFGS on the sparse operator
    res2 = si.run_adarbfgs(si.AdaConfig(prob, si.SketchRule.adaptive_cols_uniform(12), tol=0.0, max_iters=30, seed=1,
                                        track=si.TrackOptions(residual_every_k=10)))
    ref2 = O.run_adarbfgs(dense, 12, rule=O.ADA_COLS_UNIFORM, tol=0.0, max_iters=30, every_k=10, seed=1)
    assert rel(res2.state.l, ref2.x) <= ITER_TOL


def test_adarbfgs_large_q_run_parity(si):
    """q > 96 takes the Newton–Schulz inverse square root; the run must still match."""
    rng = O.RngStream(91)
    n, q = 512, 128
    a = random_spd(n, rng)
    ref = O.run_adarbfgs(a, q, rule=O.ADA_COLS_UNIFORM, tol=0.0, max_iters=12, every_k=4, seed=2)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.adaptive_cols_uniform(q),
                                       tol=0.0, max_iters=12, seed=2, track=si.TrackOptions(residual_every_k=4)))
    assert rel(res.state.l, ref.x) <= ITER_TOL


@pytest.mark.parametrize("rule", ["cols", "uniform", "gauss"])
def test_adarbfgs_step_with_caller_rng_matches_driver(si, rule):
    """adarbfgs_step (adarbfgs.cpp:49-75) advanced k times from one RngStream(seed)
    draws the same sketches as run_adarbfgs with that seed (same RNG consumption)."""
    rng0 = O.RngStream(31)
    n, q, k = 60, 6, 12
    a = random_spd(n, rng0)
    srule = {"cols": si.SketchRule.adaptive_cols(n, q), "uniform": si.SketchRule.adaptive_cols_uniform(q),
             "gauss": si.SketchRule.adaptive_gauss(q)}[rule]
    orule = {"cols": O.ADA_COLS, "uniform": O.ADA_COLS_UNIFORM, "gauss": O.ADA_GAUSS}[rule]
    prob = si.ProblemMatrix(a, si.Symmetry.spd)
    rng = si.RngStream(7)
    st = si.FactoredState(np.eye(n))
    for _ in range(k):
        st = si.adarbfgs_step(st, prob, srule, rng)
    assert st.k == k
    ref = O.run_adarbfgs(a, q, rule=orule, tol=0.0, max_iters=k, every_k=k, seed=7)
    assert rel(st.l, ref.x) <= ITER_TOL
    with pytest.raises(si.ConfigError):
        si.adarbfgs_step(st, prob, si.SketchRule.gaussian(q), rng)
