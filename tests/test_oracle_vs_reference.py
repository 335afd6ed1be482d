"""The oracle restatement (oracle/stochinv_oracle.cpp) against the reference's OWN code:
/root/reference/proj/src compiled unmodified against oracle/ref_shim into oracle/_ref
(SURVEY §8c's recommended oracle).  Trajectories — iterates, residual traces, k, the
termination and its message — of run_inverter (bfgs; Gaussian and coordinate-block
sketches), run_adarbfgs (contiguous blocks + Eq. 8.2, Gaussian S̃), the step kernels and
the sym_inv_sqrt floor decision agree to rounding, including BASELINE config 1 at full
size.  Skipped when oracle/_ref was not built (the reference tree is absent)."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")


def generators():
    """generators.py with the oracle's RngStream (byte-identical to the library's), loaded by
    path as its own module instance."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1602_01768_b200",
                        "generators.py")
    spec = importlib.util.spec_from_file_location("si_generators_ref_test", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.use_rng(O.RngStream)
    return mod


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def random_spd(n, seed):  # tests/helpers.hpp:19-22 flavour
    b = O.RngStream(seed).gaussian_matrix(n, n)
    return np.asfortranarray(b @ b.T + 0.5 * n * np.eye(n))


def traces_close(h1, h2, tol=1e-9):
    assert [h[0] for h in h1] == [h[0] for h in h2]
    r1, r2 = np.array([h[1] for h in h1]), np.array([h[1] for h in h2])
    live = r2 > 1e-12
    assert np.all(np.abs(r1[live] - r2[live]) <= tol * r2[live])
    flops1, flops2 = [h[2] for h in h1], [h[2] for h in h2]
    assert flops1 == pytest.approx(flops2, rel=1e-12)


@pytest.mark.parametrize("n,q", [(2, 1), (7, 3), (40, 5), (130, 17)])
def test_step_kernels(n, q):
    rng = O.RngStream(100 + n)
    a = random_spd(n, 200 + n)
    x = random_spd(n, 300 + n) / n
    s = rng.gaussian_matrix(n, q)
    assert rel(O.bfgs_step(x, a, s), R.bfgs_step(x, a, s)) <= 1e-12
    l = np.eye(n) + 0.1 * rng.gaussian_matrix(n, n) / np.sqrt(n)
    assert rel(O.adarbfgs_update_factor(l, a, s), R.adarbfgs_update_factor(l, a, s)) <= 1e-12


def test_bfgs_hand_fixture_on_reference():  # test_qn_updates.cpp:199-207
    a = np.array([[2.0, 1.0], [1.0, 2.0]])
    out = R.bfgs_step(np.eye(2), a, np.array([[1.0], [0.0]]))
    assert np.allclose(out, [[0.75, -0.5], [-0.5, 1.0]], atol=1e-12)
    with pytest.raises(R.RefError) as e:
        R.bfgs_step(np.eye(2), a, np.zeros((2, 1)))
    assert e.value.code == 6  # GramRankDeficientError


@pytest.mark.parametrize("ratio", [5e-15, 2e-14, 1e-13, 1e-6])
def test_sym_inv_sqrt_floor_decision(ratio):
    q = 24
    g = O.RngStream(9).gaussian_matrix(q, q)
    qm, _ = np.linalg.qr(g)
    m = (qm * np.logspace(np.log10(ratio), 0, q)) @ qm.T
    m = 0.5 * (m + m.T)
    try:
        r_ref = R.sym_inv_sqrt(m)
    except R.RefError:
        r_ref = None
    try:
        r_or = O.sym_inv_sqrt(m)
    except O.NumericalError:
        r_or = None
    assert (r_ref is None) == (r_or is None)
    if r_ref is not None:
        assert rel(r_or, r_ref) <= 1e-13 * max(1e3, 1.0 / ratio)


@pytest.mark.parametrize("rule", [O.RULE_GAUSSIAN, O.RULE_COORDINATE_BLOCK])
def test_run_inverter_trajectory(rule):
    n, q = 90, 8
    a = random_spd(n, 7)
    ro = O.run_inverter_bfgs(a, q, rule=rule, tol=0.0, max_iters=60, every_k=7, seed=4)
    rr = R.run_inverter_bfgs(a, q, rule=rule, tol=0.0, max_iters=60, every_k=7, seed=4)
    assert ro.k == rr.k == 60 and ro.termination == rr.termination
    assert rel(ro.x, rr.x) <= 1e-12
    traces_close(ro.history, rr.history)


def test_run_inverter_tolerance_and_x0():
    n, q = 48, 6
    a = random_spd(n, 8)
    x0 = np.linalg.inv(a) + 1e-3 * np.eye(n)
    x0 = 0.5 * (x0 + x0.T)
    ro = O.run_inverter_bfgs(a, q, tol=1e-6, max_iters=3000, every_k=5, seed=9, x0=x0)
    rr = R.run_inverter_bfgs(a, q, tol=1e-6, max_iters=3000, every_k=5, seed=9, x0=x0)
    assert ro.k == rr.k and ro.termination == rr.termination == 0
    assert rel(ro.x, rr.x) <= 1e-10
    traces_close(ro.history, rr.history)


def test_run_inverter_config1_full_size():
    """BASELINE config 1 (n = 1024, q = 32, Gaussian, seed 0), 50 iterations, residual every 5."""
    a = generators().config1_dense(1024, seed=0)
    ro = O.run_inverter_bfgs(a, 32, tol=0.0, max_iters=50, every_k=5, seed=0)
    rr = R.run_inverter_bfgs(a, 32, tol=0.0, max_iters=50, every_k=5, seed=0)
    assert rel(ro.x, rr.x) <= 1e-11
    traces_close(ro.history, rr.history)


@pytest.mark.parametrize("rule", ["cols", "gauss"])
def test_run_adarbfgs_trajectory(rule):
    n, q = 96, 8
    a = random_spd(n, 11)
    orule, rrule = (O.ADA_COLS, R.ADA_COLS) if rule == "cols" else (O.ADA_GAUSS, R.ADA_GAUSS)
    ro = O.run_adarbfgs(a, q, rule=orule, tol=0.0, max_iters=60, every_k=10, seed=2)
    rr = R.run_adarbfgs(a, q, rule=rrule, tol=0.0, max_iters=60, every_k=10, seed=2)
    assert ro.k == rr.k == 60
    x = ro.x @ ro.x.T  # the restatement returns L; the reference's state.x is L·Lᵀ
    assert rel(x, rr.x) <= 1e-12
    traces_close(ro.history, rr.history)


def test_run_adarbfgs_config2_shape():
    """Config 2's ridge Gram construction at n = 512 (q = 64 contiguous blocks + Eq. 8.2), 30 iterations."""
    a = generators().config2_dense(512, seed=0)
    ro = O.run_adarbfgs(a, 64, rule=O.ADA_COLS, tol=0.0, max_iters=30, every_k=10, seed=0)
    rr = R.run_adarbfgs(a, 64, rule=R.ADA_COLS, tol=0.0, max_iters=30, every_k=10, seed=0)
    assert rel(ro.x @ ro.x.T, rr.x) <= 1e-11
    traces_close(ro.history, rr.history, tol=1e-8)


def test_adarbfgs_floor_rejections_and_limit():
    """Eq. 8.2 blocks of width 2 over a matrix whose 2×2 blocks have λmin/λmax from 1e-15 to 0.35:
    the sym_inv_sqrt floor rejects some draws (redraws) — same draws, same trajectory; with
    max_redraws = 0 the first rejection ends the run (Termination::error) at the same k."""
    n, q = 16, 2
    a = np.zeros((n, n))
    deltas = [2e-15, 0.7, 1e-14, 0.5, 6e-14, 0.9, 2e-10, 0.3]
    for k in range(n // 2):
        d = deltas[k % len(deltas)]
        a[2 * k, 2 * k] = a[2 * k + 1, 2 * k + 1] = 1.0
        a[2 * k, 2 * k + 1] = a[2 * k + 1, 2 * k] = 1.0 - d
    for mr in (1000, 0):
        ro = O.run_adarbfgs(a, q, rule=O.ADA_COLS, tol=0.0, max_iters=40, every_k=10, seed=5, max_redraws=mr)
        rr = R.run_adarbfgs(a, q, rule=R.ADA_COLS, tol=0.0, max_iters=40, every_k=10, seed=5, max_redraws=mr)
        assert ro.termination == rr.termination and ro.k == rr.k
        traces_close(ro.history, rr.history, tol=1e-6)
        if mr == 0:
            assert rr.termination == 2  # Termination::error
