"""The GPU path against the reference's OWN code (oracle/_ref: /root/reference/proj/src
compiled unmodified against oracle/ref_shim; built in the development container, shipped
to the GPU box as a prebuilt library): run_inverter (bfgs) at BASELINE config 1 and
run_adarbfgs with the reference's sampler (contiguous blocks + Eq. 8.2), on the same A,
seed and host RngStream draws — iterate within 1e-9, residual trace within 1%."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")]


@pytest.fixture(scope="module")
def si():
    import paper_1602_01768_b200 as si

    return si


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_config1_run_inverter_vs_reference(si):
    from paper_1602_01768_b200 import generators as G

    a = G.config1_dense(1024, seed=0)
    ref = R.run_inverter_bfgs(a, 32, tol=0.0, max_iters=50, every_k=5, seed=0)
    res = si.run_inverter(si.InverterConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.gaussian(32), tol=0.0,
                                            max_iters=50, seed=0, track=si.TrackOptions(residual_every_k=5)))
    assert res.state.k == ref.k == 50
    assert rel(res.state.x, ref.x) <= 1e-9
    got = np.array([h.residual for h in res.state.history])
    exp = np.array([h[1] for h in ref.history])
    assert [h.k for h in res.state.history] == [h[0] for h in ref.history]
    assert np.max(np.abs(got - exp) / exp) <= 0.01
    assert res.state.flops == pytest.approx(ref.history[-1][2], rel=1e-12)  # flops.cpp tallies


def test_adarbfgs_eq82_vs_reference(si):
    b = O.RngStream(12).gaussian_matrix(256, 256)
    a = np.asfortranarray(b @ b.T / 256 + 0.5 * np.eye(256))
    ref = R.run_adarbfgs(a, 16, rule=R.ADA_COLS, tol=0.0, max_iters=60, every_k=10, seed=3)
    res = si.run_adarbfgs(si.AdaConfig(si.ProblemMatrix(a, si.Symmetry.spd), si.SketchRule.adaptive_cols(256, 16),
                                       tol=0.0, max_iters=60, seed=3, track=si.TrackOptions(residual_every_k=10)))
    assert res.state.k == ref.k == 60
    assert rel(res.state.x, ref.x) <= 1e-9  # X = L·Lᵀ (the reference's state.x)
    got = np.array([h.residual for h in res.state.history])
    exp = np.array([h[1] for h in ref.history])
    live = exp > 1e-10
    assert np.max(np.abs(got[live] - exp[live]) / exp[live]) <= 0.01
