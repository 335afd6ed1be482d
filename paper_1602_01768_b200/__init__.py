"""B200-native RBFGS / AdaRBFGS iteration (arxiv 1602.01768) behind the
reference `stochinv` solver API.

The compute path is libstochinv_b200.so (hand-written sm_100a FP64 DMMA
kernels + C ABI, include/stochinv_b200.h); this package is its Python mirror.
Importing it loads the library and raises ImportError if it is not built —
there is no CPU fallback.
"""
from . import _lib

_lib.load()

from .api import (  # noqa: E402
    AdaConfig,
    BaselineConfig,
    BaselineMethod,
    ConfigError,
    Context,
    FactoredState,
    CudaError,
    GramRankDeficientError,
    HistoryPoint,
    InverterConfig,
    InverterState,
    IoError,
    Method,
    NumericalError,
    ProbabilityRule,
    ProblemMatrix,
    RngStream,
    RunResult,
    SketchKind,
    SketchRule,
    Solver,
    Symmetry,
    Termination,
    TrackOptions,
    UpdateName,
    adaptive_block_probabilities,
    adarbfgs_step,
    aip_step,
    dfp_step,
    mr_init,
    mr_step_cached,
    newton_schulz_init,
    newton_schulz_step,
    psb_step,
    run_baseline,
    spectral_norm_estimate,
    adarbfgs_update_factor,
    sym_inv_sqrt,
    nccl_unique_id,
    bfgs_step,
    build_ridge_hessian,
    contiguous_partition,
    default_context,
    flops_adarbfgs,
    flops_bfgs,
    gen_synthetic,
    libsvm_shape,
    load_matrix_market,
    read_matrix_market,
    residual,
    run_adarbfgs,
    run_inverter,
)

__all__ = [n for n in dir() if not n.startswith("_")]
