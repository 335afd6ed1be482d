"""The other named rank-q updates (psb, aip, dfp — SURVEY §8f row f3), the
Newton–Schulz / minimal-residual baselines (row f4) and the trace harness
(row f1), on the GPU against the oracle restatements of qn_updates.cpp,
baselines.cpp and simi.cpp; harness wire-format checks run on CPU.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

ITER_TOL = 1e-9
TRACE_TOL = 0.01


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def random_spd(n, rng):  # tests/helpers.hpp:19-22
    b = rng.gaussian_matrix(n, n)
    return b @ b.T + 0.5 * n * np.eye(n)


def random_symmetric(n, rng):  # tests/helpers.hpp:24-27
    b = rng.gaussian_matrix(n, n)
    return 0.5 * (b + b.T)


def trace_gap(got, ref, floor=1e-10):
    got, ref = np.asarray(got), np.asarray(ref)
    live = ref > floor
    assert np.all(got[~live] <= 1e3 * floor)
    return float(np.max(np.abs(got[live] - ref[live]) / ref[live])) if live.any() else 0.0


@pytest.fixture(scope="module")
def si():
    import paper_1602_01768_b200 as si

    return si


# ------------------------------------------------------------ harness (CPU) --
def test_csv_wire_format(tmp_path):  # bench.cpp:167-189
    from paper_1602_01768_b200 import harness as H
    from paper_1602_01768_b200.api import HistoryPoint

    assert H.fmt(0.1) == "0.10000000000000001"
    assert H.fmt(1.0) == "1"
    assert H.fmt(2.5e-300) == "2.5e-300" and H.fmt(1.0 / 3.0) == "0.33333333333333331"
    assert H.fmt(123456789.0) == "123456789"
    t0 = H.ConvergenceTrace("bfgs", 0, [HistoryPoint(0, 1.0, 0.0, 0.0), HistoryPoint(10, 0.25, 1e9, 0.5)],
                            "max_iters")
    p = tmp_path / "one.csv"
    H.write_csv([t0], str(p))
    assert p.read_text() == ("method,iter,residual,flops,seconds\n"
                             "bfgs,0,1,0,0\n"
                             "bfgs,10,0.25,1000000000,0.5\n")
    t1 = H.ConvergenceTrace("bfgs", 1, [HistoryPoint(0, 1.0, 0.0, 0.0)], "error")
    H.write_csv([t0, t1], str(p))
    lines = p.read_text().splitlines()
    assert lines[1].startswith("bfgs#0,") and lines[3].startswith("bfgs#1,")
    svg = tmp_path / "t.svg"
    H.write_svg([t0, t1], str(svg))
    txt = svg.read_text()
    assert txt.startswith("<svg") and txt.count("<polyline") == 4 and "bfgs#1 [error]" in txt
    with pytest.raises(Exception):
        H.write_csv([t0], "/nonexistent_dir/x.csv")


def test_trial_seed_and_validation():  # bench.cpp:122-126, 141-146
    from paper_1602_01768_b200 import harness as H
    from paper_1602_01768_b200.api import ConfigError

    assert H.trial_seed(0, 0, 0) == 0x9E3779B97F4A7C15
    assert H.trial_seed(5, 1, 2) == 5 ^ ((0x9E3779B97F4A7C15 * 4099) % 2**64)
    assert H.default_q(10) == 4 and H.default_q(16) == 4 and H.default_q(1) == 1
    with pytest.raises(ConfigError):
        H.run_benchmark(None, H.BenchmarkSpec(methods=[]))
    with pytest.raises(ConfigError):
        H.run_benchmark(None, H.BenchmarkSpec(methods=[H.MethodConfig("bfgs")], tol=-1.0))
    with pytest.raises(ConfigError):
        H.run_benchmark(None, H.BenchmarkSpec(methods=[H.MethodConfig("bfgs")], trials=0))
    with pytest.raises(ConfigError, match="not on the B200 path"):
        H.run_benchmark(None, H.BenchmarkSpec(methods=[H.MethodConfig("kaczmarz")]))
    with pytest.raises(ConfigError, match="unknown update name"):
        H.run_benchmark(None, H.BenchmarkSpec(methods=[H.MethodConfig("nope")]))


# ------------------------------------------------------------ f3 step KATs --
@pytest.mark.gpu
def test_psb_aip_dfp_steps_match_oracle(si):
    rng = O.RngStream(61)
    n, q = 40, 5
    a = random_spd(n, rng)
    x = random_symmetric(n, rng)
    s = rng.gaussian_matrix(n, q)
    assert rel(si.psb_step(x, a, s), O.psb_step(x, a, s)) <= 1e-12
    assert rel(si.aip_step(x, a, s), O.aip_step(x, a, s)) <= 1e-12
    xi = O.lu_inverse(a + x @ x.T)
    xp = a + x @ x.T
    gp, gi = si.dfp_step(xp, xi, a, s)
    rp, ri = O.dfp_step(xp, xi, a, s)
    assert rel(gp, rp) <= 1e-12 and rel(gi, ri) <= 1e-11
    assert np.array_equal(gp, gp.T) and np.array_equal(gi, gi.T)


@pytest.mark.gpu
def test_psb_kkt_and_dfp_recurrence_on_gpu(si):  # test_qn_updates.cpp:119-132, 176-197
    rng = O.RngStream(23)
    a = random_symmetric(4, rng)
    x = random_symmetric(4, rng)
    s = np.zeros((4, 2))
    s[1, 0] = s[2, 1] = 1.0
    stepped = si.psb_step(x, a, s)
    assert np.linalg.norm(stepped @ a @ s - s) <= 1e-9
    rng = O.RngStream(37)
    a = random_spd(4, rng)
    full_p, full_i = si.dfp_step(np.eye(4), np.eye(4), a, np.eye(4))
    assert np.linalg.norm(full_p - a) <= 1e-9 * np.linalg.norm(a)
    assert np.linalg.norm(full_i @ a - np.eye(4)) <= 1e-8


@pytest.mark.gpu
def test_rank_deficient_sketch_raises(si):  # test_qn_updates.cpp:253-261
    rng = O.RngStream(47)
    a = random_spd(3, rng)
    for fn in (si.psb_step, si.aip_step):
        with pytest.raises(si.GramRankDeficientError):
            fn(np.eye(3), a, np.zeros((3, 1)))
    with pytest.raises(si.GramRankDeficientError):
        si.dfp_step(np.eye(3), np.eye(3), a, np.ones((3, 2)))


# ------------------------------------------------------- f3 run_inverter ----
UPD = {"psb": O.UPDATE_PSB, "aip": O.UPDATE_AIP, "dfp": O.UPDATE_DFP, "bfgs": O.UPDATE_BFGS}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["psb", "aip", "dfp"])
@pytest.mark.parametrize("rule", ["gaussian", "coord_uniform", "coord_convenient"])
def test_run_inverter_named_update_parity(si, name, rule):
    rng = O.RngStream(71)
    n, q, iters = 96, 8, 50
    a = random_spd(n, rng) / n
    orule = O.RULE_GAUSSIAN if rule == "gaussian" else O.RULE_COORDINATE_BLOCK
    oprob = O.PROB_CONVENIENT if rule == "coord_convenient" else O.PROB_UNIFORM
    ref, ref_inv = O.run_inverter(a, q, update=UPD[name], rule=orule, prob=oprob, tol=0.0, max_iters=iters,
                                  every_k=5, seed=4)
    srule = {"gaussian": si.SketchRule.gaussian(q),
             "coord_uniform": si.SketchRule.coordinate_block(n, q, si.ProbabilityRule.uniform),
             "coord_convenient": si.SketchRule.coordinate_block(n, q, si.ProbabilityRule.convenient)}[rule]
    res = si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.spd), srule, tol=0.0, max_iters=iters,
                                            seed=4, track=si.TrackOptions(residual_every_k=5), update=name))
    assert res.state.k == iters and res.termination == si.Termination.max_iters
    assert rel(res.state.x, ref.x) <= ITER_TOL
    if name == "dfp":
        assert rel(res.state.x_inv, ref_inv) <= ITER_TOL
    assert [h.k for h in res.state.history] == [h[0] for h in ref.history]
    assert trace_gap([h.residual for h in res.state.history], [h[1] for h in ref.history]) <= TRACE_TOL
    assert res.state.history[-1].flops == pytest.approx(ref.history[-1][2], rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["psb", "aip", "dfp"])
def test_run_inverter_named_update_x0_and_convergence(si, name):
    rng = O.RngStream(73)
    n, q = 48, 6
    a = random_spd(n, rng) / n
    x0 = np.eye(n) + 0.01 * random_symmetric(n, rng)
    ref, ref_inv = O.run_inverter(a, q, update=UPD[name], rule=O.RULE_GAUSSIAN, tol=1e-6, max_iters=2000,
                                  every_k=10, seed=8, x0=x0)
    res = si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.gaussian(q),
                                            tol=1e-6, max_iters=2000, seed=8, x0=x0, update=name,
                                            track=si.TrackOptions(residual_every_k=10)))
    assert res.termination == si.Termination.tol_reached == ref.termination
    assert res.state.k == ref.k
    assert rel(res.state.x, ref.x) <= 1e-7


@pytest.mark.gpu
def test_psb_requires_symmetric_and_aip_sparse_residual(si):
    rng = O.RngStream(79)
    g = rng.gaussian_matrix(8, 8) + 8 * np.eye(8)
    with pytest.raises(si.ConfigError, match="psb requires a symmetric matrix"):
        si.run_inverter(si.InverterConfig(si.ProblemMatrix(g, si.Symmetry.general), si.SketchRule.gaussian(2),
                                          update="psb"))
    # AIP iterates are not symmetric: the CSR residual goes through A·X explicitly
    from paper_1602_01768_b200 import generators as G

    n = 64
    rowptr, colind, val = G.config4_csr(n, shift=1e-1)
    sp = si.ProblemMatrix(csr=(rowptr, colind, val), n=n, symmetry=si.Symmetry.spd)
    dense = sp.data()
    ref, _ = O.run_inverter(dense, 4, update=O.UPDATE_AIP, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=30, every_k=3,
                            seed=1)
    res = si.run_inverter(si.InverterConfig(sp, si.SketchRule.gaussian(4), tol=0.0, max_iters=30, seed=1,
                                            update="aip", track=si.TrackOptions(residual_every_k=3)))
    assert rel(res.state.x, ref.x) <= ITER_TOL
    assert trace_gap([h.residual for h in res.state.history], [h[1] for h in ref.history]) <= 1e-9


# ------------------------------------------------------------- f4 baselines --
@pytest.mark.gpu
def test_baseline_building_blocks(si):  # test_baselines.cpp:14-83
    a = np.array([[2.0]])
    x = si.newton_schulz_step(np.array([[0.4]]), a)
    assert x[0, 0] == pytest.approx(0.48, rel=1e-14)
    assert si.newton_schulz_step(x, a)[0, 0] == pytest.approx(0.4992, rel=1e-14)
    assert si.newton_schulz_init(si.ProblemMatrix(a, si.Symmetry.spd))[0, 0] == pytest.approx(0.495, rel=1e-8)
    xo, _, alpha, stg = si.mr_step_cached(np.array([[0.25]]), np.eye(1) - 0.25 * a, a)
    assert xo[0, 0] == pytest.approx(0.5, rel=1e-14) and alpha == pytest.approx(2.0) and not stg
    assert np.linalg.norm(si.mr_init(si.ProblemMatrix(np.diag([1.0, 3.0]), si.Symmetry.spd)) - 0.4 * np.eye(2)) <= 1e-14
    with pytest.raises(si.ConfigError):
        si.mr_init(si.ProblemMatrix(np.zeros((2, 2)), si.Symmetry.symmetric))
    xo, _, alpha, stg = si.mr_step_cached(np.diag([0.5, 0.25]), np.zeros((2, 2)), np.diag([2.0, 4.0]))
    assert stg and alpha == 0.0 and np.array_equal(xo, np.diag([0.5, 0.25]))
    rng = O.RngStream(91)
    m = random_spd(40, rng)
    pm = si.ProblemMatrix(m, si.Symmetry.spd)
    assert si.spectral_norm_estimate(pm, 100, 3) == pytest.approx(O.spectral_norm_estimate(m, 100, 3), rel=1e-12)
    assert rel(si.newton_schulz_init(pm, 3), O.newton_schulz_init(m, 3)) <= 1e-12
    x0 = O.newton_schulz_init(m, 3)
    assert rel(si.newton_schulz_step(x0, m), O.newton_schulz_step(x0, m)) <= 1e-12
    r0 = np.eye(40) - m @ O.mr_init(m)
    g = si.mr_step_cached(O.mr_init(m), r0, m)
    o = O.mr_step_cached(O.mr_init(m), r0, m)
    assert rel(g[0], o[0]) <= 1e-12 and rel(g[1], o[1]) <= 1e-11 and g[2] == pytest.approx(o[2], rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["newton_schulz", "minimal_residual"])
def test_run_baseline_parity(si, method):
    rng = O.RngStream(97)
    n = 120
    a = random_spd(n, rng)
    om = O.BASELINE_NS if method == "newton_schulz" else O.BASELINE_MR
    iters = 40 if method == "newton_schulz" else 60
    ref = O.run_baseline(a, method=om, tol=0.0, max_iters=iters, every_k=5, seed=2)
    res = si.run_baseline(si.BaselineConfig(si.ProblemMatrix(a, si.Symmetry.spd), method=si.BaselineMethod[method],
                                            tol=0.0, max_iters=iters, seed=2,
                                            track=si.TrackOptions(residual_every_k=5)))
    assert res.termination == si.Termination(ref.termination)
    assert [h.k for h in res.state.history] == [h[0] for h in ref.history]
    assert trace_gap([h.residual for h in res.state.history], [h[1] for h in ref.history], floor=1e-12) <= 1e-6
    assert rel(res.state.x, ref.x) <= 1e-9
    assert [h.flops for h in res.state.history] == [h[2] for h in ref.history]


@pytest.mark.gpu
def test_run_baseline_contract(si):  # test_baselines.cpp:85-146
    rng = O.RngStream(97)
    a = random_spd(12, rng)
    pm = si.ProblemMatrix(a, si.Symmetry.spd)
    ns = si.run_baseline(si.BaselineConfig(pm, tol=1e-8, max_iters=200, track=si.TrackOptions(residual_every_k=5)))
    assert ns.termination == si.Termination.tol_reached
    assert np.linalg.norm(a @ ns.state.x - np.eye(12)) <= 1e-6 * np.linalg.norm(a)
    assert ns.state.history[0].residual == 1.0 and ns.state.flops > 0
    mr = si.run_baseline(si.BaselineConfig(pm, method=si.BaselineMethod.minimal_residual, tol=1e-2, max_iters=5000,
                                           track=si.TrackOptions(residual_every_k=25)))
    assert mr.termination == si.Termination.tol_reached and mr.state.history[-1].residual <= 1e-2
    stiff = si.ProblemMatrix(random_spd(10, O.RngStream(101)), si.Symmetry.spd)
    div = si.run_baseline(si.BaselineConfig(stiff, x0=np.eye(10), max_iters=200))
    assert div.termination == si.Termination.error and "diverged" in div.message
    with pytest.raises(si.ConfigError):
        si.run_baseline(si.BaselineConfig(pm, tol=-1.0))
    exact = si.run_baseline(si.BaselineConfig(si.ProblemMatrix(np.diag([2.0, 4.0]), si.Symmetry.spd),
                                              x0=np.diag([0.5, 0.25])))
    assert exact.termination == si.Termination.tol_reached and exact.state.history[0].residual == 0.0


# ---------------------------------------------------------- f1 harness GPU --
@pytest.mark.gpu
def test_run_benchmark_traces_match_oracle_and_are_deterministic(si, tmp_path):
    from paper_1602_01768_b200 import harness as H

    a_prob = H.MatrixSource(H.MatrixSourceKind.synthetic, n=30, seed=3).load()
    a = a_prob.data()
    methods = [H.MethodConfig("bfgs", q=3), H.MethodConfig("psb", q=3), H.MethodConfig("aip", q=3),
               H.MethodConfig("dfp", q=3, probabilities=si.ProbabilityRule.convenient),
               H.MethodConfig("adarbfgs-cols", q=3), H.MethodConfig("newton-schulz"), H.MethodConfig("mr")]
    spec = H.BenchmarkSpec(methods=methods, tol=1e-12, max_iters=60, seed=11, trials=2, residual_every_k=10,
                           measure_time=False)
    traces = H.run_benchmark(a_prob, spec)
    assert [(t.method, t.trial) for t in traces] == [(m.name, t) for m in methods for t in range(2)]
    for i, tr in enumerate(traces):
        mi, t = divmod(i, 2)
        seed = H.trial_seed(11, mi, t)
        name = tr.method
        if name in ("bfgs", "psb", "aip", "dfp"):
            prob = O.PROB_CONVENIENT if name == "dfp" else O.PROB_UNIFORM
            ref, _ = O.run_inverter(a, 3, update=UPD[name], rule=O.RULE_COORDINATE_BLOCK, prob=prob, tol=1e-12,
                                    max_iters=60, every_k=10, seed=seed)
        elif name == "adarbfgs-cols":
            ref = O.run_adarbfgs(a, 3, rule=O.ADA_COLS, tol=1e-12, max_iters=60, every_k=10, seed=seed)
        else:
            ref = O.run_baseline(a, method=O.BASELINE_NS if name == "newton-schulz" else O.BASELINE_MR, tol=1e-12,
                                 max_iters=60, every_k=10, seed=seed)
        assert [p.k for p in tr.points] == [h[0] for h in ref.history], name
        assert trace_gap([p.residual for p in tr.points], [h[1] for h in ref.history], floor=1e-9) <= TRACE_TOL, name
        assert all(p.seconds == 0.0 for p in tr.points)
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    H.write_csv(traces, str(p1))
    H.write_csv(H.run_benchmark(a_prob, spec), str(p2))
    assert p1.read_bytes() == p2.read_bytes()  # measure_time=False: byte-identical CSVs (bench.hpp:49)
    assert p1.read_text().splitlines()[0] == "method,iter,residual,flops,seconds"
