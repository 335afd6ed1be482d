"""Multi-GPU C ABI (shard.cpp) on the GPU: the sharded RBFGS / AdaRBFGS drivers behind
si_run_inverter / si_run_adarbfgs / si_solver_* on multi-GPU contexts.

One GPU is available to the tests, so the P > 1 logic runs on the loopback context
(P virtual ranks on one device, collectives replayed as device copies — every chunk /
panel, exchange, all-gather and all-reduce of the sharded iteration is exercised with
uneven partitions), and the NCCL paths at P = 1 (ncclCommInitAll over one device, and a
one-process-per-GPU group of size 1), both with the iterations replayed as CUDA graphs
with the collectives captured.  Everything is compared with the single-GPU driver (same
A, seed and sketches) and with the CPU oracle: iterate within 1e-9 relative Frobenius,
residual trace within 1%, drawn coordinates bit-exact.
Reference: proj/src/simi.cpp:217-381, proj/src/adarbfgs.cpp:91-200 (run semantics).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-9
TRACE_TOL = 0.01


@pytest.fixture(scope="module")
def si():
    import paper_1602_01768_b200 as si

    return si


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def random_spd(n, seed):
    b = O.RngStream(seed).gaussian_matrix(n, n)
    return np.asfortranarray(b @ b.T / n + 0.5 * np.eye(n))


def traces(res):
    return [h.k for h in res.state.history], np.array([h.residual for h in res.state.history])


def trace_gap(got, ref, floor=1e-10):
    """Max relative gap over the points above the rounding floor (below it — finite
    termination at machine precision — both must be tiny)."""
    got, ref = np.asarray(got), np.asarray(ref)
    live = ref > floor
    assert np.all(got[~live] <= 1e3 * floor)
    return float(np.max(np.abs(got[live] - ref[live]) / ref[live])) if live.any() else 0.0


def contexts(si, kind, P):
    if kind == "loopback":
        return si.Context.loopback(0, P)
    if kind == "multi":
        return si.Context.multi([0])
    return si.Context.rank(0, 1, 0, si.nccl_unique_id())


def run_rbfgs(si, ctx, a, q, rule, iters, every, seed, csr=None):
    n = a.shape[0]
    prob = (si.ProblemMatrix(csr=csr, n=n, symmetry=si.Symmetry.spd, context=ctx) if csr is not None else
            si.ProblemMatrix(a, si.Symmetry.spd, context=ctx))
    return si.run_inverter(si.InverterConfig(prob, rule, tol=0.0, max_iters=iters, seed=seed,
                                             track=si.TrackOptions(residual_every_k=every)))


@pytest.mark.parametrize("kind,P", [("loopback", 1), ("loopback", 2), ("loopback", 3), ("multi", 1), ("rank", 1)])
def test_rbfgs_sharded_device_sketch_matches_single(si, kind, P):
    """Batched device-sketch loop (graph replays incl. the collectives) against the single-GPU driver."""
    n, q, iters, every, seed = 301, 16, 30, 10, 5
    a = random_spd(n, 11)
    ref = run_rbfgs(si, si.Context(0), a, q, si.SketchRule.gaussian_device(q), iters, every, seed)
    ctx = contexts(si, kind, P)
    assert ctx.ranks()[0] == P
    got = run_rbfgs(si, ctx, a, q, si.SketchRule.gaussian_device(q), iters, every, seed)
    assert got.state.k == ref.state.k == iters
    assert rel(got.state.x, ref.state.x) <= ITER_TOL
    assert np.array_equal(got.state.x, got.state.x.T)
    kg, tg = traces(got)
    kr, tr = traces(ref)
    assert kg == kr
    assert trace_gap(tg, tr) <= TRACE_TOL
    assert got.state.flops == pytest.approx(ref.state.flops)


@pytest.mark.parametrize("P", [2, 3])
def test_rbfgs_sharded_host_sketch_matches_oracle(si, P):
    n, q, iters, every, seed = 200, 12, 25, 5, 3
    a = random_spd(n, 21)
    ref = O.run_inverter_bfgs(a, q, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=iters, every_k=every, seed=seed)
    got = run_rbfgs(si, si.Context.loopback(0, P), a, q, si.SketchRule.gaussian(q), iters, every, seed)
    assert rel(got.state.x, ref.x) <= ITER_TOL
    kg, tg = traces(got)
    assert kg == [h[0] for h in ref.history]
    assert trace_gap(tg, [h[1] for h in ref.history]) <= TRACE_TOL


def test_rbfgs_sharded_coordinate_block_draws(si):
    n, q, iters, seed = 90, 8, 40, 9  # ragged partition: the last block is 2 wide
    a = random_spd(n, 31)
    ref = O.run_inverter_bfgs(a, q, rule=O.RULE_COORDINATE_BLOCK, tol=0.0, max_iters=iters, every_k=10, seed=seed)
    ctx = si.Context.loopback(0, 3)
    ctx.set_draw_log(4 * iters)
    got = run_rbfgs(si, ctx, a, q, si.SketchRule.coordinate_block(n, q), iters, 10, seed)
    assert rel(got.state.x, ref.x) <= ITER_TOL
    single = si.Context(0)
    single.set_draw_log(4 * iters)
    run_rbfgs(si, single, a, q, si.SketchRule.coordinate_block(n, q), iters, 10, seed)
    assert np.array_equal(ctx.draw_log(), single.draw_log()) and ctx.draw_log().size == iters


@pytest.mark.parametrize("P", [1, 3])
def test_rbfgs_sharded_csr(si, P):
    from paper_1602_01768_b200 import generators as G

    n, q, iters, seed = 400, 24, 20, 2
    rp, ci, va = G.config5_csr(n, half_bandwidth=6, seed=1)
    dense = G.csr_to_dense(n, rp, ci, va)
    ref = run_rbfgs(si, si.Context(0), dense, q, si.SketchRule.gaussian_device(q), iters, 10, seed, csr=(rp, ci, va))
    got = run_rbfgs(si, si.Context.loopback(0, P), dense, q, si.SketchRule.gaussian_device(q), iters, 10, seed,
                    csr=(rp, ci, va))
    assert rel(got.state.x, ref.state.x) <= ITER_TOL
    assert trace_gap(traces(got)[1], traces(ref)[1]) <= TRACE_TOL


def test_rbfgs_sharded_x0_and_errors(si):
    n, q = 120, 8
    a = random_spd(n, 41)
    x0 = np.asfortranarray(np.linalg.inv(a) + 0.01 * np.eye(n))
    x0 = 0.5 * (x0 + x0.T)
    ref = O.run_inverter_bfgs(a, q, rule=O.RULE_GAUSSIAN, tol=0.0, max_iters=10, every_k=5, seed=1, x0=x0)
    ctx = si.Context.loopback(0, 2)
    prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
    got = si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(q), tol=0.0, max_iters=10, seed=1, x0=x0,
                                            track=si.TrackOptions(residual_every_k=5)))
    assert rel(got.state.x, ref.x) <= ITER_TOL
    assert abs(got.state.history[-1].residual - ref.history[-1][1]) <= 1e-2 * ref.history[-1][1]
    bad = a.copy()
    bad[0, 0] = -1.0
    # validate_spd: "spd flag set but Cholesky failed" is a plain std::runtime_error in the reference
    # (problem_matrix.cpp:36-40), which the C ABI maps like the CLI does (exit 2: ConfigError)
    with pytest.raises((si.ConfigError, si.NumericalError)):
        si.run_inverter(si.InverterConfig(si.ProblemMatrix(bad, si.Symmetry.spd, context=ctx),
                                          si.SketchRule.gaussian(q), max_iters=2))
    with pytest.raises(si.ConfigError):
        si.run_inverter(si.InverterConfig(prob, si.SketchRule.gaussian(q), update=si.UpdateName.psb, max_iters=2))


@pytest.mark.parametrize("kind,P", [("loopback", 1), ("loopback", 2), ("loopback", 3), ("multi", 1)])
@pytest.mark.parametrize("rule", ["uniform", "cols", "gauss"])
def test_adarbfgs_sharded_matches_oracle(si, kind, P, rule):
    n, q, iters, every, seed = 97, 8, 40, 10, 4  # uneven panels (97 = 33 + 32 + 32)
    a = random_spd(n, 51)
    orule = {"uniform": O.ADA_COLS_UNIFORM, "cols": O.ADA_COLS, "gauss": O.ADA_GAUSS}[rule]
    ref = O.run_adarbfgs(a, q, rule=orule, tol=0.0, max_iters=iters, every_k=every, seed=seed)
    ctx = contexts(si, kind, P)
    ctx.set_draw_log(iters * q * 4)
    srule = {"uniform": si.SketchRule.adaptive_cols_uniform(q), "cols": si.SketchRule.adaptive_cols(n, q),
             "gauss": si.SketchRule.adaptive_gauss(q)}[rule]
    got = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd, context=ctx), srule, tol=0.0,
                                       max_iters=iters, seed=seed, track=si.TrackOptions(residual_every_k=every)))
    assert got.state.k == iters
    assert rel(got.state.l, ref.x) <= ITER_TOL
    assert rel(got.state.x, got.state.l @ got.state.l.T) <= 1e-12
    kg, tg = traces(got)
    rt = np.array([h[1] for h in ref.history])
    assert kg == [h[0] for h in ref.history]
    assert trace_gap(tg, rt) <= TRACE_TOL
    if rule != "gauss":
        drawn = ctx.draw_log()
        assert drawn.size > 0 and np.array_equal(drawn, ref.outcomes[:drawn.size])


def test_adarbfgs_sharded_device_gauss_and_csr(si):
    from paper_1602_01768_b200 import generators as G

    n, q, iters, seed = 144, 16, 20, 6
    rp, ci, va = G.config4_csr(n)
    dense = G.csr_to_dense(n, rp, ci, va)
    for rule in (si.SketchRule.adaptive_gauss_device(q), si.SketchRule.adaptive_cols_uniform(q)):
        runs = []
        for ctx in (si.Context(0), si.Context.loopback(0, 3)):
            prob = si.ProblemMatrix(csr=(rp, ci, va), n=n, symmetry=si.Symmetry.spd, context=ctx)
            runs.append(si.run_adarbfgs(si.AdaConfig(prob, rule, tol=0.0, max_iters=iters, seed=seed,
                                                     track=si.TrackOptions(residual_every_k=10))))
        assert rel(runs[1].state.l, runs[0].state.l) <= ITER_TOL
        assert trace_gap(traces(runs[1])[1], traces(runs[0])[1]) <= TRACE_TOL
    assert np.isfinite(dense).all()


def test_adarbfgs_sharded_l0_eq82(si):
    n, q, iters, seed = 64, 8, 30, 2
    a = random_spd(n, 61)
    l0 = np.eye(n) + 0.01 * O.RngStream(3).gaussian_matrix(n, n)
    ref = O.run_adarbfgs(a, q, rule=O.ADA_COLS, tol=0.0, max_iters=iters, every_k=10, seed=seed, l0=l0)
    ctx = si.Context.loopback(0, 2)
    got = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd, context=ctx),
                                       si.SketchRule.adaptive_cols(n, q), tol=0.0, max_iters=iters, seed=seed, l0=l0,
                                       track=si.TrackOptions(residual_every_k=10)))
    assert rel(got.state.l, ref.x) <= ITER_TOL


@pytest.mark.parametrize("P", [1, 2, 3])
def test_sharded_solver_matches_single(si, P):
    n, q, seed = 260, 16, 8
    a = random_spd(n, 71)
    out = []
    for ctx in (si.Context(0), si.Context.loopback(0, P)):
        prob = si.ProblemMatrix(a, si.Symmetry.spd, context=ctx)
        s = si.Solver(prob, si.Method.rbfgs, si.SketchRule.gaussian_device(q), seed=seed)
        s.step(7)
        s.step(5)
        out.append((s.iterate(), s.residual()))
    assert rel(out[1][0], out[0][0]) <= ITER_TOL
    assert out[1][1] == pytest.approx(out[0][1], rel=1e-8)
