"""TEST INFRASTRUCTURE — ctypes access to oracle/_ref/libstochinv_ref.so: the reference's OWN
sources (/root/reference/proj/src, unmodified) compiled against oracle/ref_shim (a
from-scratch Eigen-API subset over OpenBLAS) by `make -C oracle ref`.  Used by the tests to
pin the oracle restatement to the reference code itself, and by bench.py's reference arm.
Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs load it.

`available()` is False when the library was not built (no /root/reference at build time).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .oracle import RunResult  # same result shape as the restatement's drivers

_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_DIR, "_ref", "libstochinv_ref.so")
REF_ROOT = "/root/reference/proj"
_lib = None

RULE_GAUSSIAN, RULE_COORDINATE_BLOCK = 0, 1
ADA_COLS, ADA_GAUSS = 0, 1


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build() -> bool:
    """Compile oracle/_ref when the reference tree is present (this container)."""
    if not os.path.isdir(REF_ROOT):
        return os.path.exists(LIB_PATH)
    subprocess.run(["make", "-C", _DIR, "ref"], check=True, capture_output=True)
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{LIB_PATH} is not built (make -C oracle ref, needs {REF_ROOT})")
        L = C.CDLL(LIB_PATH)
        pd, pi64, i64, u64 = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int64, C.c_uint64
        L.rf_last_error.restype = C.c_char_p
        L.rf_bfgs_step.argtypes = [i64, i64, pd, pd, pd, pd]
        L.rf_adarbfgs_update_factor.argtypes = [i64, i64, pd, pd, pd, pd]
        L.rf_sym_inv_sqrt.argtypes = [i64, pd, pd]
        L.rf_run_inverter_bfgs.argtypes = [i64, pd, C.c_int, i64, C.c_double, i64, i64, u64, C.c_int, pd, pd,
                                           C.POINTER(C.c_int), pi64, pi64, pd, pd, pd, i64, pi64, pd, C.c_char_p, i64]
        L.rf_run_adarbfgs.argtypes = [i64, pd, C.c_int, i64, C.c_double, i64, i64, u64, C.c_int, pd, pd,
                                      C.POINTER(C.c_int), pi64, pi64, pd, pd, pd, i64, pi64]
        _lib = L
    return _lib


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().rf_last_error().decode())


def bfgs_step(x, a, s) -> np.ndarray:  # qn_updates.cpp:176-186
    x, a, s = _f(x), _f(a), _f(s)
    out = np.empty_like(x, order="F")
    _check(lib().rf_bfgs_step(x.shape[0], s.shape[1], _p(x), _p(a), _p(s), _p(out)))
    return out


def adarbfgs_update_factor(l, a, st) -> np.ndarray:  # adarbfgs.cpp:12-21
    l, a, st = _f(l), _f(a), _f(st)
    out = np.empty_like(l, order="F")
    _check(lib().rf_adarbfgs_update_factor(l.shape[0], st.shape[1], _p(l), _p(a), _p(st), _p(out)))
    return out


def sym_inv_sqrt(m) -> np.ndarray:  # linalg.cpp:144-155
    m = _f(m)
    out = np.empty_like(m, order="F")
    _check(lib().rf_sym_inv_sqrt(m.shape[0], _p(m), _p(out)))
    return out


def _history(hk, hr, hf, hs, count, cap):
    m = min(count, cap)
    return [(int(hk[i]), float(hr[i]), float(hf[i]), float(hs[i])) for i in range(m)]


def run_inverter_bfgs(a, q, *, rule=RULE_GAUSSIAN, tol=1e-2, max_iters=1000, every_k=10, seed=0, max_redraws=100,
                      x0=None, want_x=True) -> RunResult:
    """The reference's run_inverter (simi.cpp:217-381) for MethodSpec::named_method(bfgs)."""
    a = _f(a)
    n = a.shape[0]
    xo = np.empty((n, n), order="F") if want_x else None
    x0f = _f(x0) if x0 is not None else None
    cap = max_iters + 2
    hk = np.zeros(cap, dtype=np.int64)
    hr, hf, hs = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    term, k, hc, drift = C.c_int(), C.c_int64(), C.c_int64(), C.c_double()
    msg = C.create_string_buffer(512)
    _check(lib().rf_run_inverter_bfgs(n, _p(a), rule, q, tol, max_iters, every_k, seed, max_redraws, _p(x0f), _p(xo),
                                      C.byref(term), C.byref(k), hk.ctypes.data_as(C.POINTER(C.c_int64)), _p(hr),
                                      _p(hf), _p(hs), cap, C.byref(hc), C.byref(drift), msg, 512))
    r = RunResult(xo, term.value, k.value, _history(hk, hr, hf, hs, hc.value, cap), drift.value)
    r.message = msg.value.decode()
    return r


def run_adarbfgs(a, q, *, rule=ADA_COLS, tol=1e-2, max_iters=1000, every_k=10, seed=0, max_redraws=100,
                 l0=None) -> RunResult:
    """The reference's run_adarbfgs (adarbfgs.cpp:91-200); `x` is state.x = L·Lᵀ."""
    a = _f(a)
    n = a.shape[0]
    xo = np.empty((n, n), order="F")
    l0f = _f(l0) if l0 is not None else None
    cap = max_iters + 2
    hk = np.zeros(cap, dtype=np.int64)
    hr, hf, hs = np.zeros(cap), np.zeros(cap), np.zeros(cap)
    term, k, hc = C.c_int(), C.c_int64(), C.c_int64()
    _check(lib().rf_run_adarbfgs(n, _p(a), rule, q, tol, max_iters, every_k, seed, max_redraws, _p(l0f), _p(xo),
                                 C.byref(term), C.byref(k), hk.ctypes.data_as(C.POINTER(C.c_int64)), _p(hr), _p(hf),
                                 _p(hs), cap, C.byref(hc)))
    return RunResult(xo, term.value, k.value, _history(hk, hr, hf, hs, hc.value, cap))
