"""Golden vectors produced by the reference's own code (tests/golden/make_golden.py, through
oracle/_ref) pin both the oracle restatement (CPU) and the CUDA path (GPU): step kernels,
sym_inv_sqrt, run_inverter (Gaussian and coordinate-block sketches) and run_adarbfgs
(contiguous blocks + Eq. 8.2 and Gaussian S̃) — checkpoint schedule and flop tallies equal,
iterate within 1e-9 relative Frobenius, residual trace within 1% (north-star bars)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz"))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def check_trace(hist, prefix, tol=0.01):
    hk, hr, hf = GOLD[prefix + "_hk"], GOLD[prefix + "_hr"], GOLD[prefix + "_hf"]
    assert [h[0] for h in hist] == list(hk)
    got = np.array([h[1] for h in hist])
    live = hr > 1e-10
    assert np.max(np.abs(got[live] - hr[live]) / hr[live]) <= tol
    np.testing.assert_allclose([h[2] for h in hist], hf, rtol=1e-12)  # flops.cpp tallies


# ------------------------------------------------------------------ oracle (CPU)
def test_oracle_step_kernels_match_reference_vectors():
    out = O.bfgs_step(GOLD["step_x"], GOLD["step_a"], GOLD["step_s"])
    assert rel(out, GOLD["step_bfgs_out"]) <= 1e-12
    out = O.adarbfgs_update_factor(GOLD["step_l"], GOLD["step_a"], GOLD["step_st"])
    assert rel(out, GOLD["step_ada_out"]) <= 1e-12
    assert rel(O.sym_inv_sqrt(GOLD["isqrt_m"]), GOLD["isqrt_out"]) <= 1e-12


@pytest.mark.parametrize("name,rule,seed", [("run_gauss", O.RULE_GAUSSIAN, 3), ("run_coord", O.RULE_COORDINATE_BLOCK, 5)])
def test_oracle_run_inverter_matches_reference_vectors(name, rule, seed):
    r = O.run_inverter_bfgs(GOLD["run_a"], 6, rule=rule, tol=0.0, max_iters=30, every_k=5, seed=seed)
    assert r.k == 30
    assert rel(r.x, GOLD[name + "_x"]) <= 1e-11
    check_trace(r.history, name, tol=1e-9)


@pytest.mark.parametrize("name,rule,seed", [("ada_cols", O.ADA_COLS, 3), ("ada_gauss", O.ADA_GAUSS, 9)])
def test_oracle_run_adarbfgs_matches_reference_vectors(name, rule, seed):
    r = O.run_adarbfgs(GOLD["ada_a"], 8, rule=rule, tol=0.0, max_iters=40, every_k=10, seed=seed)
    assert r.k == 40
    assert rel(r.x @ r.x.T, GOLD[name + "_x"]) <= 1e-11  # the oracle returns L, the reference X = L·Lᵀ
    check_trace(r.history, name, tol=1e-8)


# --------------------------------------------------------------------- CUDA path
@pytest.fixture(scope="module")
def si():
    import paper_1602_01768_b200 as si

    return si


@pytest.mark.gpu
def test_gpu_step_kernels_match_reference_vectors(si):
    out = si.bfgs_step(GOLD["step_x"], GOLD["step_a"], GOLD["step_s"])
    assert rel(out, GOLD["step_bfgs_out"]) <= 1e-11
    out = si.adarbfgs_update_factor(GOLD["step_l"], GOLD["step_a"], GOLD["step_st"])
    assert rel(out, GOLD["step_ada_out"]) <= 1e-11
    assert rel(si.sym_inv_sqrt(GOLD["isqrt_m"]), GOLD["isqrt_out"]) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed", [("run_gauss", 3), ("run_coord", 5)])
def test_gpu_run_inverter_matches_reference_vectors(si, name, seed):
    a = GOLD["run_a"]
    rule = si.SketchRule.gaussian(6) if name == "run_gauss" else si.SketchRule.coordinate_block(48, 6)
    res = si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.spd), rule, tol=0.0, max_iters=30,
                                            seed=seed, track=si.TrackOptions(residual_every_k=5)))
    assert res.state.k == 30
    assert rel(res.state.x, GOLD[name + "_x"]) <= 1e-9
    check_trace([(h.k, h.residual, h.flops) for h in res.state.history], name)


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed", [("ada_cols", 3), ("ada_gauss", 9)])
def test_gpu_run_adarbfgs_matches_reference_vectors(si, name, seed):
    a = GOLD["ada_a"]
    rule = si.SketchRule.adaptive_cols(64, 8) if name == "ada_cols" else si.SketchRule.adaptive_gauss(8)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), rule, tol=0.0, max_iters=40, seed=seed,
                                       track=si.TrackOptions(residual_every_k=10)))
    assert res.state.k == 40
    assert rel(res.state.x, GOLD[name + "_x"]) <= 1e-9
    check_trace([(h.k, h.residual, h.flops) for h in res.state.history], name)
