"""ctypes binding of the CPU oracle — TEST INFRASTRUCTURE ONLY.

The oracle (`oracle/stochinv_oracle.cpp`) is a C++ restatement of the
reference's RBFGS / AdaRBFGS hot path (see its header).  This module is imported
only by tests/, `__graft_entry__.smoke()` and bench.py's CPU-baseline legs, as
the checker; the product package never imports it.

All matrices are numpy float64 arrays in Fortran (column-major) order, the
layout of Eigen::MatrixXd in the reference (proj/include/stochinv/types.hpp:8).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")

_d = C.c_double
_i64 = C.c_int64
_pd = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)


def build() -> str:
    subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def _load():
    if not os.path.exists(_LIB_PATH):
        build()
    lib = C.CDLL(_LIB_PATH)
    lib.or_last_error.restype = C.c_char_p
    lib.or_rng_create.restype = C.c_void_p
    lib.or_rng_create.argtypes = [C.c_uint64]
    lib.or_rng_substream.restype = C.c_void_p
    lib.or_rng_substream.argtypes = [C.c_void_p, C.c_uint64]
    lib.or_rng_destroy.argtypes = [C.c_void_p]
    lib.or_rng_uniform.restype = _d
    lib.or_rng_uniform.argtypes = [C.c_void_p]
    lib.or_rng_gaussian.restype = _d
    lib.or_rng_gaussian.argtypes = [C.c_void_p]
    lib.or_rng_categorical.restype = _i64
    lib.or_rng_categorical.argtypes = [C.c_void_p, _pd, _i64]
    lib.or_rng_uniform_index.restype = _i64
    lib.or_rng_uniform_index.argtypes = [C.c_void_p, _i64]
    lib.or_rng_gaussian_matrix.argtypes = [C.c_void_p, _i64, _i64, _pd]
    lib.or_rng_uniform_matrix.argtypes = [C.c_void_p, _i64, _i64, _pd]
    lib.or_uniform_subset.argtypes = [C.c_void_p, _i64, _i64, _pi64]
    lib.or_bfgs_step.argtypes = [_i64, _i64, _pd, _pd, _pd, _pd]
    lib.or_symmetrize.restype = _d
    lib.or_symmetrize.argtypes = [_i64, _pd]
    lib.or_adarbfgs_update_factor.argtypes = [_i64, _i64, _pd, _pd, _pd, _pd]
    lib.or_adaptive_block_probabilities.argtypes = [_i64, _i64, _pd, _pd, _pd]
    lib.or_sym_inv_sqrt.argtypes = [_i64, _pd, _pd]
    lib.or_jacobi.argtypes = [_i64, _pd, _pd, _pd]
    lib.or_gemm.argtypes = [_i64, _i64, _i64, C.c_int, C.c_int, _pd, _pd, _pd]
    lib.or_residual.restype = _d
    lib.or_residual.argtypes = [_i64, _pd, _pd]
    lib.or_flops_bfgs.restype = _d
    lib.or_flops_bfgs.argtypes = [_i64, _i64]
    lib.or_flops_adarbfgs.restype = _d
    lib.or_flops_adarbfgs.argtypes = [_i64, _i64]
    lib.or_have_blas.restype = C.c_int
    lib.or_run_inverter_bfgs.argtypes = [
        _i64, _pd, C.c_int, _i64, _d, _i64, _i64, C.c_uint64, C.c_int, _pd, _pd,
        C.POINTER(C.c_int), _pi64, _pi64, _pd, _pd, _pd, _i64, _pi64, _pd, _pi64]
    lib.or_run_adarbfgs.argtypes = [
        _i64, _pd, C.c_int, _i64, _d, _i64, _i64, C.c_uint64, C.c_int, _pd, _pd,
        C.POINTER(C.c_int), _pi64, _pi64, _pd, _pd, _pd, _i64, _pi64, _pi64, _i64]
    lib.or_set_threads.argtypes = [C.c_int]
    lib.or_psb_step.argtypes = [_i64, _i64, _pd, _pd, _pd, _pd]
    lib.or_aip_step.argtypes = [_i64, _i64, _pd, _pd, _pd, _pd]
    lib.or_dfp_step.argtypes = [_i64, _i64, _pd, _pd, _pd, _pd, _pd, _pd]
    lib.or_lu_inverse.argtypes = [_i64, _pd, _pd]
    lib.or_flops_named.restype = _d
    lib.or_flops_named.argtypes = [C.c_int, _i64, _i64]
    lib.or_newton_schulz_step.argtypes = [_i64, _pd, _pd, _pd]
    lib.or_newton_schulz_init.argtypes = [_i64, _pd, C.c_uint64, _pd]
    lib.or_spectral_norm_estimate.argtypes = [_i64, _i64, _pd, C.c_int, C.c_uint64, _pd]
    lib.or_mr_step_cached.argtypes = [_i64, _pd, _pd, _pd, _pd, _pd, _pd, C.POINTER(C.c_int)]
    lib.or_mr_init.argtypes = [_i64, _pd, _pd]
    lib.or_run_baseline.argtypes = [
        _i64, _pd, C.c_int, _d, _i64, _i64, C.c_uint64, _pd, _pd, C.POINTER(C.c_int), _pi64, _pi64, _pd, _pd,
        _pd, _i64, _pi64]
    lib.or_run_inverter.argtypes = [
        C.c_int, _i64, _pd, C.c_int, C.c_int, _i64, _d, _i64, _i64, C.c_uint64, C.c_int, _pd, _pd, _pd,
        C.POINTER(C.c_int), _pi64, _pi64, _pd, _pd, _pd, _i64, _pi64, _pd, _pi64]
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(OracleError, ValueError):
    pass


class NumericalError(OracleError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().or_last_error().decode()
    if rc == 2:
        raise ConfigError(rc, msg)
    if rc == 3:
        raise NumericalError(rc, msg)
    raise OracleError(rc, msg)


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_pd)


class RngStream:
    """rng.hpp:13-71 restated (the same std::mt19937_64 + libstdc++ distributions)."""

    def __init__(self, seed: int = 0, _handle=None):
        self._h = _handle if _handle is not None else lib().or_rng_create(C.c_uint64(seed & (2**64 - 1)))

    def __del__(self):
        try:
            if self._h:
                lib().or_rng_destroy(self._h)
        except Exception:
            pass

    def substream(self, index: int) -> "RngStream":
        return RngStream(_handle=lib().or_rng_substream(self._h, C.c_uint64(index)))

    def uniform(self) -> float:
        return lib().or_rng_uniform(self._h)

    def gaussian(self) -> float:
        return lib().or_rng_gaussian(self._h)

    def categorical(self, p) -> int:
        p = np.ascontiguousarray(p, dtype=np.float64)
        return int(lib().or_rng_categorical(self._h, _p(p), p.size))

    def uniform_index(self, n: int) -> int:
        return int(lib().or_rng_uniform_index(self._h, n))

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        lib().or_rng_gaussian_matrix(self._h, rows, cols, _p(out))
        return out

    def uniform_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64, order="F")
        lib().or_rng_uniform_matrix(self._h, rows, cols, _p(out))
        return out

    def uniform_subset(self, n: int, q: int) -> np.ndarray:
        out = np.empty(q, dtype=np.int64)
        lib().or_uniform_subset(self._h, n, q, out.ctypes.data_as(_pi64))
        return out


def bfgs_step(x, a, s) -> np.ndarray:
    """qn_updates.cpp:176-186."""
    x, a, s = _f(x), _f(a), _f(s)
    n, q = s.shape
    out = np.empty((n, n), order="F")
    _check(lib().or_bfgs_step(n, q, _p(x), _p(a), _p(s), _p(out)))
    return out


def symmetrize_(x: np.ndarray) -> float:
    """In place X = (X + Xᵀ)/2, returns the removed drift ‖X − Xᵀ‖_F (simi.cpp:351-357)."""
    assert x.flags.f_contiguous and x.dtype == np.float64
    return float(lib().or_symmetrize(x.shape[0], _p(x)))


def adarbfgs_update_factor(l, a, stilde) -> np.ndarray:
    """adarbfgs.cpp:12-21."""
    l, a, st = _f(l), _f(a), _f(stilde)
    n, q = st.shape
    out = np.empty((n, n), order="F")
    _check(lib().or_adarbfgs_update_factor(n, q, _p(l), _p(a), _p(st), _p(out)))
    return out


def adaptive_block_probabilities(l, a, q: int) -> np.ndarray:
    """adarbfgs.cpp:23-36 over contiguous_partition(n, q) (sketching.cpp:106-115)."""
    l, a = _f(l), _f(a)
    n = l.shape[0]
    nb = (n + q - 1) // q
    out = np.empty(nb)
    _check(lib().or_adaptive_block_probabilities(n, q, _p(l), _p(a), _p(out)))
    return out


def sym_inv_sqrt(m) -> np.ndarray:
    m = _f(m)
    out = np.empty_like(m, order="F")
    _check(lib().or_sym_inv_sqrt(m.shape[0], _p(m), _p(out)))
    return out


def jacobi_eigendecomposition(m):
    m = _f(m)
    n = m.shape[0]
    vals = np.empty(n)
    vecs = np.empty((n, n), order="F")
    _check(lib().or_jacobi(n, _p(m), _p(vals), _p(vecs)))
    return vals, vecs


def residual(a, x) -> float:
    """‖I − A X‖_F (simi.cpp:242-244)."""
    a, x = _f(a), _f(x)
    return float(lib().or_residual(a.shape[0], _p(a), _p(x)))


def flops_bfgs(n, q) -> float:
    return float(lib().or_flops_bfgs(n, q))


def flops_adarbfgs(n, q) -> float:
    return float(lib().or_flops_adarbfgs(n, q))


def set_threads(n: int) -> None:
    """Host threads for OpenBLAS and the elementwise passes (0 = all)."""
    lib().or_set_threads(int(n))


def have_blas() -> bool:
    return bool(lib().or_have_blas())


@dataclass
class RunResult:
    x: np.ndarray
    termination: int
    k: int
    history: list = field(default_factory=list)  # (k, residual, flops, seconds)
    max_symmetry_drift: float = 0.0
    redraws: int = 0
    outcomes: np.ndarray | None = None


RULE_GAUSSIAN, RULE_COORDINATE_BLOCK = 0, 1
ADA_COLS, ADA_GAUSS, ADA_COLS_UNIFORM = 0, 1, 2


def run_inverter_bfgs(a, q, *, rule=RULE_GAUSSIAN, tol=1e-2, max_iters=1000, every_k=10, seed=0,
                      max_redraws=100, x0=None) -> RunResult:
    """run_inverter for MethodSpec::named_method(bfgs) (simi.cpp:217-381)."""
    a = _f(a)
    n = a.shape[0]
    xo = np.empty((n, n), order="F")
    x0p = _p(_f(x0)) if x0 is not None else None
    if x0 is not None:
        x0f = _f(x0)
        x0p = _p(x0f)
    cap = max_iters + 2
    hk = np.zeros(cap, dtype=np.int64)
    hr, hf, hs = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    term, k, hc, red = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
    drift = C.c_double()
    _check(lib().or_run_inverter_bfgs(n, _p(a), rule, q, tol, max_iters, every_k, seed, max_redraws, x0p, _p(xo),
                                      C.byref(term), C.byref(k), hk.ctypes.data_as(_pi64), _p(hr), _p(hf), _p(hs),
                                      cap, C.byref(hc), C.byref(drift), C.byref(red)))
    m = min(hc.value, cap)
    hist = [(int(hk[i]), float(hr[i]), float(hf[i]), float(hs[i])) for i in range(m)]
    return RunResult(xo, term.value, k.value, hist, drift.value, red.value)


def run_adarbfgs(a, q, *, rule=ADA_COLS, tol=1e-2, max_iters=1000, every_k=10, seed=0, max_redraws=100,
                 l0=None, max_outcomes=None) -> RunResult:
    """run_adarbfgs (adarbfgs.cpp:91-200); rule ADA_COLS_UNIFORM is the paper sampler."""
    a = _f(a)
    n = a.shape[0]
    lo = np.empty((n, n), order="F")
    l0p = None
    if l0 is not None:
        l0f = _f(l0)
        l0p = _p(l0f)
    cap = max_iters + 2
    hk = np.zeros(cap, dtype=np.int64)
    hr, hf, hs = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    ocap = max_outcomes or max_iters * (q if rule == ADA_COLS_UNIFORM else 1) * 2 + 16
    outc = np.zeros(ocap, dtype=np.int64)
    term, k, hc = C.c_int(), C.c_int64(), C.c_int64()
    _check(lib().or_run_adarbfgs(n, _p(a), rule, q, tol, max_iters, every_k, seed, max_redraws, l0p, _p(lo),
                                 C.byref(term), C.byref(k), hk.ctypes.data_as(_pi64), _p(hr), _p(hf), _p(hs), cap,
                                 C.byref(hc), outc.ctypes.data_as(_pi64), ocap))
    m = min(hc.value, cap)
    hist = [(int(hk[i]), float(hr[i]), float(hf[i]), float(hs[i])) for i in range(m)]
    return RunResult(lo, term.value, k.value, hist, outcomes=outc)


# ------------------------------------------------ row f3: other updates --
UPDATE_BFGS, UPDATE_PSB, UPDATE_AIP, UPDATE_DFP = 0, 1, 2, 3
PROB_UNIFORM, PROB_CONVENIENT = 0, 1


def psb_step(x, a, s) -> np.ndarray:  # qn_updates.cpp:121-129
    x, a, s = _f(x), _f(a), _f(s)
    o = np.empty_like(x, order="F")
    _check(lib().or_psb_step(x.shape[0], s.shape[1], _p(x), _p(a), _p(s), _p(o)))
    return o


def aip_step(x, a, s) -> np.ndarray:  # qn_updates.cpp:147-152
    x, a, s = _f(x), _f(a), _f(s)
    o = np.empty_like(x, order="F")
    _check(lib().or_aip_step(x.shape[0], s.shape[1], _p(x), _p(a), _p(s), _p(o)))
    return o


def dfp_step(x, x_inv, a, s):  # qn_updates.cpp:154-174 -> (primal, inverse)
    x, xi, a, s = _f(x), _f(x_inv), _f(a), _f(s)
    o, oi = np.empty_like(x, order="F"), np.empty_like(x, order="F")
    _check(lib().or_dfp_step(x.shape[0], s.shape[1], _p(x), _p(xi), _p(a), _p(s), _p(o), _p(oi)))
    return o, oi


def lu_inverse(m) -> np.ndarray:  # linalg.cpp:157-160
    m = _f(m)
    o = np.empty_like(m, order="F")
    _check(lib().or_lu_inverse(m.shape[0], _p(m), _p(o)))
    return o


def flops_named(update: int, n: int, q: int) -> float:
    return float(lib().or_flops_named(update, n, q))


def run_inverter(a, q, *, update=UPDATE_BFGS, rule=RULE_GAUSSIAN, prob=PROB_UNIFORM, tol=1e-2, max_iters=1000,
                 every_k=10, seed=0, max_redraws=100, x0=None):
    """run_inverter for MethodSpec::named_method(bfgs|psb|aip|dfp) (simi.cpp:217-381).
    Returns (RunResult, x_inv) with x_inv the tracked inverse for dfp (else None)."""
    a = _f(a)
    n = a.shape[0]
    xo = np.empty((n, n), order="F")
    xio = np.empty((n, n), order="F") if update == UPDATE_DFP else None
    x0f = _f(x0) if x0 is not None else None
    cap = max_iters + 2
    hk = np.zeros(cap, dtype=np.int64)
    hr, hf, hs = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    term, k, hc, red = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
    drift = C.c_double()
    _check(lib().or_run_inverter(update, n, _p(a), rule, prob, q, tol, max_iters, every_k, seed, max_redraws,
                                 _p(x0f) if x0f is not None else None, _p(xo),
                                 _p(xio) if xio is not None else None, C.byref(term), C.byref(k),
                                 hk.ctypes.data_as(_pi64), _p(hr), _p(hf), _p(hs), cap, C.byref(hc), C.byref(drift),
                                 C.byref(red)))
    m = min(hc.value, cap)
    hist = [(int(hk[i]), float(hr[i]), float(hf[i]), float(hs[i])) for i in range(m)]
    return RunResult(xo, term.value, k.value, hist, drift.value, red.value), xio


# ------------------------------------------------ row f4: baselines --
BASELINE_NS, BASELINE_MR = 0, 1


def newton_schulz_step(x, a) -> np.ndarray:  # baselines.cpp:12-14
    x, a = _f(x), _f(a)
    o = np.empty_like(x, order="F")
    _check(lib().or_newton_schulz_step(x.shape[0], _p(x), _p(a), _p(o)))
    return o


def newton_schulz_init(a, seed=0) -> np.ndarray:  # baselines.cpp:16-20
    a = _f(a)
    o = np.empty_like(a, order="F")
    _check(lib().or_newton_schulz_init(a.shape[0], _p(a), seed, _p(o)))
    return o


def spectral_norm_estimate(m, iters=100, seed=0) -> float:  # linalg.cpp:106-129
    m = _f(m)
    est = C.c_double()
    _check(lib().or_spectral_norm_estimate(m.shape[0], m.shape[1], _p(m), iters, seed, C.byref(est)))
    return est.value


def mr_step_cached(x, r, a):  # baselines.cpp:22-37 -> (x, r, alpha, stagnated)
    x, r, a = _f(x), _f(r), _f(a)
    xo, ro = np.empty_like(x, order="F"), np.empty_like(x, order="F")
    al, stg = C.c_double(), C.c_int()
    _check(lib().or_mr_step_cached(x.shape[0], _p(x), _p(r), _p(a), _p(xo), _p(ro), C.byref(al), C.byref(stg)))
    return xo, ro, al.value, bool(stg.value)


def mr_init(a) -> np.ndarray:  # baselines.cpp:45-50
    a = _f(a)
    o = np.empty_like(a, order="F")
    _check(lib().or_mr_init(a.shape[0], _p(a), _p(o)))
    return o


def run_baseline(a, *, method=BASELINE_NS, tol=1e-2, max_iters=1000, every_k=10, seed=0, x0=None) -> RunResult:
    """run_baseline (baselines.cpp:52-151)."""
    a = _f(a)
    n = a.shape[0]
    xo = np.empty((n, n), order="F")
    x0f = _f(x0) if x0 is not None else None
    cap = max_iters + 2
    hk = np.zeros(cap, dtype=np.int64)
    hr, hf, hs = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    term, k, hc = C.c_int(), C.c_int64(), C.c_int64()
    _check(lib().or_run_baseline(n, _p(a), method, tol, max_iters, every_k, seed,
                                 _p(x0f) if x0f is not None else None, _p(xo), C.byref(term), C.byref(k),
                                 hk.ctypes.data_as(_pi64), _p(hr), _p(hf), _p(hs), cap, C.byref(hc)))
    m = min(hc.value, cap)
    hist = [(int(hk[i]), float(hr[i]), float(hf[i]), float(hs[i])) for i in range(m)]
    return RunResult(xo, term.value, k.value, hist)
