"""ctypes binding of libstochinv_b200.so (the C ABI in include/stochinv_b200.h).

Loading fails loudly when the library has not been built: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libstochinv_b200.so")

d, i64, u64, ci = C.c_double, C.c_int64, C.c_uint64, C.c_int
pd, pi64, pi32, vp = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_void_p

CHECKPOINT_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class HistoryPoint(C.Structure):
    _fields_ = [("k", i64), ("residual", d), ("flops", d), ("seconds", d)]


class InverterConfigC(C.Structure):
    _fields_ = [
        ("sketch", ci), ("probabilities", ci), ("q", i64), ("tol", d), ("max_iters", i64),
        ("time_budget_seconds", d), ("seed", u64), ("residual_every_k", i64), ("track_flops", ci),
        ("track_wall_time", ci), ("max_redraws", ci), ("x0_host", pd), ("on_checkpoint", CHECKPOINT_FN),
        ("user", vp), ("update", ci),
    ]


class RunResultC(C.Structure):
    _fields_ = [
        ("termination", ci), ("k", i64), ("max_symmetry_drift", d), ("flops", d), ("seconds", d),
        ("history_count", i64), ("redraws", i64), ("condition_estimate", d), ("message", C.c_char * 256),
    ]


_SIGS = {
    "si_last_error": (C.c_char_p, []),
    "si_version": (C.c_char_p, []),
    "si_default_config": (None, [C.POINTER(InverterConfigC)]),
    "si_context_create": (ci, [ci, C.POINTER(vp)]),
    "si_context_create_on_stream": (ci, [ci, vp, C.POINTER(vp)]),
    "si_context_destroy": (ci, [vp]),
    "si_context_synchronize": (ci, [vp]),
    "si_context_release_workspaces": (ci, [vp]),
    "si_context_launch_count": (i64, [vp]),
    "si_context_set_draw_log": (ci, [vp, pi64, i64]),
    "si_nccl_unique_id": (ci, [vp]),
    "si_context_create_multi": (ci, [C.POINTER(ci), ci, C.POINTER(vp)]),
    "si_context_create_rank": (ci, [ci, vp, ci, ci, vp, C.POINTER(vp)]),
    "si_context_create_loopback": (ci, [ci, ci, C.POINTER(vp)]),
    "si_context_ranks": (ci, [vp, C.POINTER(ci), C.POINTER(ci), C.POINTER(ci)]),
    "si_sym_inv_sqrt": (ci, [vp, i64, pd, pd]),
    "si_context_draw_count": (i64, [vp]),
    "si_context_set_profiling": (ci, [vp, ci]),
    "si_context_profile": (ci, [vp, vp, pi64, pd, ci]),
    "si_context_reset_profile": (ci, [vp]),
    "si_problem_create_dense": (ci, [vp, i64, pd, ci, C.POINTER(vp)]),
    "si_problem_create_dense_device": (ci, [vp, i64, vp, ci, C.POINTER(vp)]),
    "si_problem_create_csr": (ci, [vp, i64, i64, pi64, pi32, pd, ci, C.POINTER(vp)]),
    "si_problem_destroy": (ci, [vp]),
    "si_problem_n": (i64, [vp]),
    "si_problem_validate_spd": (ci, [vp]),
    "si_problem_get_dense": (ci, [vp, pd]),
    "si_problem_load_matrix_market": (ci, [vp, C.c_char_p, ci, ci, C.POINTER(vp)]),
    "si_problem_ridge_hessian": (ci, [vp, C.c_char_p, d, C.POINTER(vp)]),
    "si_problem_synthetic": (ci, [vp, i64, u64, C.POINTER(vp)]),
    "si_io_matrix_market_info": (ci, [C.c_char_p, pi64, C.POINTER(ci), pi64]),
    "si_io_matrix_market_dense": (ci, [C.c_char_p, pd]),
    "si_io_libsvm_info": (ci, [C.c_char_p, pi64, pi64]),
    "si_bfgs_step": (ci, [vp, i64, i64, pd, pd, pd, pd]),
    "si_bfgs_step_problem": (ci, [vp, vp, i64, pd, pd, pd]),
    "si_adarbfgs_update_factor": (ci, [vp, i64, i64, pd, pd, pd, pd]),
    "si_adaptive_block_probabilities": (ci, [vp, i64, pd, pd, i64, pi64, pi64, pd]),
    "si_residual": (ci, [vp, vp, pd, pd]),
    "si_run_inverter": (ci, [vp, vp, C.POINTER(InverterConfigC), pd, C.POINTER(HistoryPoint), i64,
                             C.POINTER(RunResultC)]),
    "si_run_inverter_pair": (ci, [vp, vp, C.POINTER(InverterConfigC), pd, pd, C.POINTER(HistoryPoint), i64,
                                  C.POINTER(RunResultC)]),
    "si_run_baseline": (ci, [vp, vp, ci, C.POINTER(InverterConfigC), pd, C.POINTER(HistoryPoint), i64,
                             C.POINTER(RunResultC)]),
    "si_psb_step": (ci, [vp, i64, i64, pd, pd, pd, pd]),
    "si_aip_step": (ci, [vp, i64, i64, pd, pd, pd, pd]),
    "si_dfp_step": (ci, [vp, i64, i64, pd, pd, pd, pd, pd, pd]),
    "si_newton_schulz_step": (ci, [vp, i64, pd, pd, pd]),
    "si_newton_schulz_init": (ci, [vp, vp, u64, pd]),
    "si_spectral_norm_estimate": (ci, [vp, vp, ci, u64, pd]),
    "si_mr_step_cached": (ci, [vp, i64, pd, pd, pd, pd, pd, pd, C.POINTER(ci)]),
    "si_mr_init": (ci, [vp, vp, pd]),
    "si_run_adarbfgs": (ci, [vp, vp, C.POINTER(InverterConfigC), pd, pd, C.POINTER(HistoryPoint), i64,
                             C.POINTER(RunResultC)]),
    "si_solver_create": (ci, [vp, vp, ci, ci, i64, u64, C.POINTER(vp)]),
    "si_solver_destroy": (ci, [vp]),
    "si_solver_set_identity": (ci, [vp]),
    "si_solver_set_iterate": (ci, [vp, pd]),
    "si_solver_get_iterate": (ci, [vp, pd]),
    "si_solver_iterate_device": (vp, [vp]),
    "si_solver_step": (ci, [vp, i64]),
    "si_solver_step_with_sketch": (ci, [vp, pd, pi64]),
    "si_solver_residual": (ci, [vp, pd]),
    "si_solver_redraws": (i64, [vp]),
    "si_gemm_device": (ci, [vp, i64, i64, i64, vp, i64, ci, vp, i64, ci, vp, i64, d, d]),
    "si_spmm_csr_device": (ci, [vp, i64, i64, vp, vp, vp, vp, i64, i64, vp, i64]),
    "si_symupd_device": (ci, [vp, i64, i64, vp, i64, vp, i64, vp, i64]),
    "si_sketch_gaussian_device": (ci, [vp, vp, i64, i64, i64, u64, u64]),
    "si_rbfgs_core_device": (ci, [vp, vp, i64, i64, vp, vp]),
    "si_rbfgs_core_device_async": (ci, [vp, vp, i64, i64, vp, vp, vp]),
    "si_gather_columns_device": (ci, [vp, vp, i64, i64, vp, i64, vp]),
    "si_ada_core_device": (ci, [vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, vp]),
    "si_pdiag_update_device": (ci, [vp, vp, i64, i64, vp, vp, vp]),
    "si_residual_rows_device": (ci, [vp, vp, i64, i64, vp, i64, pd]),
    "si_problem_dense_device": (vp, [vp]),
    "si_adarbfgs_step": (ci, [vp, vp, ci, i64, vp, ci, pd, pd]),
    "si_rng_create": (ci, [u64, C.POINTER(vp)]),
    "si_rng_substream": (ci, [vp, u64, C.POINTER(vp)]),
    "si_rng_destroy": (ci, [vp]),
    "si_rng_uniform": (d, [vp]),
    "si_rng_gaussian": (d, [vp]),
    "si_rng_categorical": (i64, [vp, pd, i64]),
    "si_rng_uniform_index": (i64, [vp, i64]),
    "si_rng_gaussian_matrix": (ci, [vp, i64, i64, pd]),
    "si_rng_uniform_matrix": (ci, [vp, i64, i64, pd]),
    "si_rng_uniform_subset": (ci, [vp, i64, i64, pi64]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1602_01768_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
