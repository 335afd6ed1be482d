"""Generate tests/golden/reference_vectors.npz from the reference's OWN code.

Run in the development container, where /root/reference exists:

    python -c "import __graft_entry__ as g; g.build()"     # builds oracle/_ref from /root/reference/proj/src
    python tests/golden/make_golden.py

Every output below is produced by oracle/_ref/libstochinv_ref.so — the reference's sources
(qn_updates.cpp, adarbfgs.cpp, linalg.cpp, simi.cpp, sketching.cpp, ...) compiled unmodified
against oracle/ref_shim — through oracle/ref.py.  The inputs are seeded numpy draws, stored
next to the outputs.  The fixtures pin the oracle restatement (CPU tests) and the CUDA path
(GPU tests) to the reference even where oracle/_ref itself is not available.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref as R  # noqa: E402


def spd(n, seed, shift=0.5):
    b = np.random.default_rng(seed).standard_normal((n, n))
    return np.asfortranarray(b @ b.T / n + shift * np.eye(n))


def hist(r):
    return (np.array([h[0] for h in r.history], dtype=np.int64), np.array([h[1] for h in r.history]),
            np.array([h[2] for h in r.history]))


def main():
    if not R.available():
        raise SystemExit("oracle/_ref is not built (needs /root/reference)")
    out = {}
    rng = np.random.default_rng(2024)
    # --- step kernels: bfgs_step (qn_updates.cpp:176-186), adarbfgs_update_factor (adarbfgs.cpp:12-21)
    n, q = 24, 4
    a = spd(n, 1)
    x = rng.standard_normal((n, n))
    x = np.asfortranarray((x + x.T) / 2)
    s = np.asfortranarray(rng.standard_normal((n, q)))
    out["step_a"], out["step_x"], out["step_s"] = a, x, s
    out["step_bfgs_out"] = R.bfgs_step(x, a, s)
    l = np.asfortranarray(np.eye(n) + 0.1 * rng.standard_normal((n, n)))
    st = np.asfortranarray(rng.standard_normal((n, q)))
    out["step_l"], out["step_st"] = l, st
    out["step_ada_out"] = R.adarbfgs_update_factor(l, a, st)
    # --- sym_inv_sqrt (linalg.cpp:144-155)
    m = spd(8, 7, shift=0.1)
    out["isqrt_m"] = m
    out["isqrt_out"] = R.sym_inv_sqrt(m)
    # --- run_inverter, named bfgs (simi.cpp:217-381): Gaussian and coordinate-block sketches
    a = spd(48, 3)
    out["run_a"] = a
    r = R.run_inverter_bfgs(a, 6, rule=R.RULE_GAUSSIAN, tol=0.0, max_iters=30, every_k=5, seed=3)
    out["run_gauss_x"] = r.x
    out["run_gauss_hk"], out["run_gauss_hr"], out["run_gauss_hf"] = hist(r)
    r = R.run_inverter_bfgs(a, 6, rule=R.RULE_COORDINATE_BLOCK, tol=0.0, max_iters=30, every_k=5, seed=5)
    out["run_coord_x"] = r.x
    out["run_coord_hk"], out["run_coord_hr"], out["run_coord_hf"] = hist(r)
    # --- run_adarbfgs (adarbfgs.cpp:91-200): contiguous blocks + Eq. 8.2, and Gaussian S̃
    a = spd(64, 4)
    out["ada_a"] = a
    r = R.run_adarbfgs(a, 8, rule=R.ADA_COLS, tol=0.0, max_iters=40, every_k=10, seed=3)
    out["ada_cols_x"] = r.x
    out["ada_cols_hk"], out["ada_cols_hr"], out["ada_cols_hf"] = hist(r)
    r = R.run_adarbfgs(a, 8, rule=R.ADA_GAUSS, tol=0.0, max_iters=40, every_k=10, seed=9)
    out["ada_gauss_x"] = r.x
    out["ada_gauss_hk"], out["ada_gauss_hr"], out["ada_gauss_hf"] = hist(r)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes;", len(out), "arrays")


if __name__ == "__main__":
    main()
