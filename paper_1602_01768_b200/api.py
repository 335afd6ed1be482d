"""Python mirror of the reference's solver API, backed by the sm_100a C ABI.

Names, argument meaning and error behaviour follow proj/include/stochinv/
(qn_updates.hpp:70 bfgs_step, adarbfgs.hpp:28-59, simi.hpp:38-107,
sketching.hpp:37-77, problem_matrix.hpp:7-35, rng.hpp:13-71, errors.hpp:9-26)
so tests and callers read like the reference's own.  Every matrix computation
runs on the GPU through libstochinv_b200.so; matrices cross the boundary as
column-major float64 host arrays (numpy, order="F"), Eigen::MatrixXd's layout.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib as L

# ----------------------------------------------------------------- errors --


class StochinvError(Exception):
    code = 5


class ConfigError(StochinvError, ValueError):  # errors.hpp:9-12
    code = 2


class NumericalError(StochinvError, RuntimeError):  # errors.hpp:14-17
    code = 3


class GramRankDeficientError(NumericalError):  # errors.hpp:19-22 (resample signal)
    code = 6


class IoError(StochinvError, OSError):  # errors.hpp:24-26
    code = 4


class CudaError(StochinvError, RuntimeError):
    code = 5


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = L.load().si_last_error().decode(errors="replace")
    cls = {2: ConfigError, 3: NumericalError, 4: IoError, 5: CudaError, 6: GramRankDeficientError}.get(rc, StochinvError)
    raise cls(msg)


def _f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _pd(a: np.ndarray):
    return a.ctypes.data_as(L.pd)


# ---------------------------------------------------------------- context --


class Context:
    """One device context (stream, workspaces); owned by one host thread.

    Multi-GPU contexts (the sharded drivers, shard.cpp) come from the class methods
    `multi(devices)` (one process, several GPUs), `rank(device, nranks, rank, nccl_id)`
    (one process per GPU, torchrun style; rank 0 makes the id with nccl_unique_id()) and
    `loopback(device, nranks)` (virtual ranks on one GPU: a test harness)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, *, _handle=None):
        lib = L.load()
        if _handle is not None:
            h = _handle
        else:
            h = C.c_void_p()
            if stream is None:
                _check(lib.si_context_create(device, C.byref(h)))
            else:
                _check(lib.si_context_create_on_stream(device, C.c_void_p(stream), C.byref(h)))
        self._h = h
        self.device = device
        # the CUDA stream the context launches on when the caller chose it (None: the
        # context's private stream); dist.CudaPanelOps requires torch's current stream here
        self.stream = stream

    @classmethod
    def multi(cls, devices: Sequence[int]) -> "Context":
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(L.load().si_context_create_multi(arr, len(devices), C.byref(h)))
        return cls(devices[0], _handle=h)

    @classmethod
    def rank(cls, device: int, nranks: int, rank: int, nccl_id: bytes, stream: Optional[int] = None) -> "Context":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
        _check(L.load().si_context_create_rank(device, C.c_void_p(stream) if stream else None, nranks, rank, buf,
                                               C.byref(h)))
        ctx = cls(device, _handle=h)
        ctx.stream = stream
        return ctx

    @classmethod
    def loopback(cls, device: int, nranks: int) -> "Context":
        h = C.c_void_p()
        _check(L.load().si_context_create_loopback(device, nranks, C.byref(h)))
        return cls(device, _handle=h)

    def ranks(self):
        """(global rank count, global rank of the first local rank, local rank count)."""
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        _check(L.load().si_context_ranks(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        _check(L.load().si_context_synchronize(self._h))

    def launch_count(self) -> int:
        return int(L.load().si_context_launch_count(self._h))

    def set_draw_log(self, cap: int) -> None:
        """Record the drivers' sampling outcomes (block indices / uniform coordinates, every
        executed attempt in draw order) from now on; read them with draw_log()."""
        self._draw_buf = np.zeros(max(int(cap), 1), dtype=np.int64) if cap else None
        buf = self._draw_buf
        _check(L.load().si_context_set_draw_log(self._h, buf.ctypes.data_as(L.pi64) if buf is not None else None,
                                                 int(cap)))

    def draw_log(self) -> np.ndarray:
        cnt = int(L.load().si_context_draw_count(self._h))
        buf = getattr(self, "_draw_buf", None)
        if buf is None:
            return np.zeros(0, dtype=np.int64)
        if cnt > buf.size:
            raise RuntimeError(f"draw log overflow: {cnt} entries, capacity {buf.size}")
        return buf[:cnt].copy()

    def release_workspaces(self):
        """Free the run_inverter / run_adarbfgs workspace the context keeps between calls."""
        _check(L.load().si_context_release_workspaces(self._h))

    def set_profiling(self, on: bool):
        _check(L.load().si_context_set_profiling(self._h, 1 if on else 0))

    def reset_profile(self):
        _check(L.load().si_context_reset_profile(self._h))

    def profile(self) -> dict:
        cap = 64
        names = (C.c_char * 32 * cap)()
        launches = (C.c_int64 * cap)()
        ms = (C.c_double * cap)()
        cnt = L.load().si_context_profile(self._h, names, launches, ms, cap)
        if cnt < 0:
            _check(-cnt)
        return {bytes(names[i]).split(b"\0")[0].decode(): (int(launches[i]), float(ms[i])) for i in range(min(cnt, cap))}

    def close(self):
        if getattr(self, "_h", None):
            L.load().si_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


NCCL_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId on this process (rank 0 of a one-process-per-GPU group)."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(L.load().si_nccl_unique_id(buf))
    return buf.raw


_tls = threading.local()


def default_context() -> Context:
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(0)
        _tls.ctx = ctx
    return ctx


# ------------------------------------------------------------ core types ---


class Symmetry(enum.IntEnum):  # problem_matrix.hpp:7
    general = 0
    symmetric = 1
    spd = 2


class ProbabilityRule(enum.IntEnum):  # sketching.hpp:24-31 (subset used by bfgs)
    uniform = 0
    convenient = 1
    none = 9


class SketchKind(enum.IntEnum):  # si_sketch_kind
    gaussian_dense = 0
    gaussian_device = 1
    coordinate_block = 2
    adaptive_factor_cols = 3
    adaptive_factor_gauss = 4
    adaptive_factor_cols_uniform = 5
    adaptive_factor_gauss_device = 6


class UpdateName(enum.IntEnum):  # qn_updates.hpp UpdateName, the members on the B200 path (si_update)
    bfgs = 0
    psb = 1
    aip = 2
    dfp = 3

    @classmethod
    def _missing_(cls, value):  # update_name_from_string (qn_updates.cpp:55-65) for the CLI vocabulary
        if isinstance(value, str):
            for m in cls:
                if m.name == value:
                    return m
            raise ConfigError(f"unknown update name: {value}")
        return None


class BaselineMethod(enum.IntEnum):  # baselines.hpp:36
    newton_schulz = 0
    minimal_residual = 1


class Termination(enum.IntEnum):  # simi.hpp:80
    tol_reached = 0
    max_iters = 1
    error = 2


class ProblemMatrix:
    """ProblemMatrix(Matrix, Symmetry) (problem_matrix.hpp:12-35), resident on the GPU.

    Dense input is symmetrized (M + Mᵀ)/2 for symmetric/spd flags as the
    reference does (problem_matrix.cpp:9-18).  `csr=(rowptr, colind, val)`
    builds a sparse A instead (configs 4/5; the reference densifies)."""

    def __init__(self, data=None, symmetry: Symmetry = Symmetry.spd, *, csr=None, n: Optional[int] = None,
                 context: Optional[Context] = None):
        self.ctx = context or default_context()
        lib = L.load()
        h = C.c_void_p()
        self.symmetry = Symmetry(symmetry)
        if csr is not None:
            rowptr, colind, val = csr
            rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
            colind = np.ascontiguousarray(colind, dtype=np.int32)
            val = np.ascontiguousarray(val, dtype=np.float64)
            n = int(n if n is not None else rowptr.size - 1)
            _check(lib.si_problem_create_csr(self.ctx.handle, n, int(val.size), rowptr.ctypes.data_as(L.pi64),
                                             colind.ctypes.data_as(L.pi32), _pd(val), int(symmetry), C.byref(h)))
            self.sparse = True
            self.nnz = int(val.size)
        else:
            a = _f64(data)
            if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < 1:
                raise ConfigError("ProblemMatrix: matrix must be square with n >= 1")
            n = a.shape[0]
            _check(lib.si_problem_create_dense(self.ctx.handle, n, _pd(a), int(symmetry), C.byref(h)))
            self.sparse = False
            self.nnz = n * n
        self._h = h
        self._n = int(n)

    def n(self) -> int:
        return self._n

    @property
    def handle(self):
        return self._h

    def is_symmetric(self) -> bool:
        return self.symmetry != Symmetry.general

    def validate_spd(self) -> None:
        _check(L.load().si_problem_validate_spd(self._h))

    def data(self) -> np.ndarray:
        out = np.empty((self._n, self._n), order="F")
        _check(L.load().si_problem_get_dense(self._h, _pd(out)))
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                L.load().si_problem_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _problem_from_handle(h, ctx, symmetry) -> ProblemMatrix:
    pm = ProblemMatrix.__new__(ProblemMatrix)
    pm.ctx = ctx
    pm._h = h
    pm._n = int(L.load().si_problem_n(h))
    pm.symmetry = Symmetry(symmetry)
    pm.sparse = L.load().si_problem_dense_device(h) is None
    pm.nnz = pm._n * pm._n if not pm.sparse else -1
    return pm


def load_matrix_market(path: str, symmetry: Optional[Symmetry] = None, keep_sparse: bool = True,
                       context: Optional[Context] = None) -> ProblemMatrix:
    """ProblemMatrix load_matrix_market(path) (io.hpp:14): header checks, line-numbered
    IoError; coordinate files stay CSR when keep_sparse (the reference densifies)."""
    ctx = context or default_context()
    h = C.c_void_p()
    sym = -1 if symmetry is None else int(symmetry)
    _check(L.load().si_problem_load_matrix_market(ctx.handle, str(path).encode(), sym, 1 if keep_sparse else 0,
                                                  C.byref(h)))
    if symmetry is None:
        # the header decides (general / symmetric); read it back from the file banner
        with open(path) as f:
            symmetry = Symmetry.symmetric if "symmetric" in f.readline().lower() else Symmetry.general
    return _problem_from_handle(h, ctx, symmetry)


def build_ridge_hessian(path: str, lam: float, context: Optional[Context] = None) -> ProblemMatrix:
    """ProblemMatrix build_ridge_hessian(path, lambda) (io.hpp:19): BᵀB + λI on the GPU."""
    ctx = context or default_context()
    h = C.c_void_p()
    _check(L.load().si_problem_ridge_hessian(ctx.handle, str(path).encode(), float(lam), C.byref(h)))
    return _problem_from_handle(h, ctx, Symmetry.spd if lam > 0 else Symmetry.symmetric)


def gen_synthetic(n: int, seed: int = 0, context: Optional[Context] = None) -> ProblemMatrix:
    """ProblemMatrix gen_synthetic(n, seed) (io.hpp:23): ĀᵀĀ with Ā ~ U(0,1) from RngStream(seed)."""
    ctx = context or default_context()
    h = C.c_void_p()
    _check(L.load().si_problem_synthetic(ctx.handle, int(n), C.c_uint64(seed), C.byref(h)))
    return _problem_from_handle(h, ctx, Symmetry.spd)


def read_matrix_market(path: str) -> tuple[np.ndarray, bool]:
    """Host parse of a MatrixMarket file: (dense n×n, header-symmetric) — what the
    reference's load_matrix_market(path).data() holds (io.cpp:28-121), no device work."""
    lib = L.load()
    n, sym, stored = C.c_int64(), C.c_int(), C.c_int64()
    _check(lib.si_io_matrix_market_info(str(path).encode(), C.byref(n), C.byref(sym), C.byref(stored)))
    out = np.zeros((n.value, n.value), dtype=np.float64, order="F")
    _check(lib.si_io_matrix_market_dense(str(path).encode(), _pd(out)))
    return out, bool(sym.value)


def libsvm_shape(path: str) -> tuple[int, int]:
    """(samples, features) of a LIBSVM file, with the reference's parse errors (io.cpp:128-161)."""
    m, n = C.c_int64(), C.c_int64()
    _check(L.load().si_io_libsvm_info(str(path).encode(), C.byref(m), C.byref(n)))
    return m.value, n.value


def contiguous_partition(n: int, q: int) -> list[list[int]]:  # sketching.cpp:106-115
    if q < 1 or q > n:
        raise ConfigError("contiguous_partition: need 1 <= q <= n")
    return [list(range(s, min(s + q, n))) for s in range(0, n, q)]


@dataclass
class SketchRule:  # sketching.hpp:37-69 (the subset on the hot path)
    kind: SketchKind = SketchKind.gaussian_dense
    q: int = 1
    probabilities: ProbabilityRule = ProbabilityRule.none
    blocks: list = field(default_factory=list)

    @staticmethod
    def gaussian(q: int) -> "SketchRule":
        return SketchRule(SketchKind.gaussian_dense, q, ProbabilityRule.none)

    @staticmethod
    def gaussian_device(q: int) -> "SketchRule":
        """Gaussian S from the device counter-based RNG (perf mode; not bit-parity)."""
        return SketchRule(SketchKind.gaussian_device, q, ProbabilityRule.none)

    @staticmethod
    def coordinate_block(n: int, q: int, prob: ProbabilityRule = ProbabilityRule.uniform) -> "SketchRule":
        return SketchRule(SketchKind.coordinate_block, q, prob, contiguous_partition(n, q))

    @staticmethod
    def adaptive_cols(n: int, q: int) -> "SketchRule":
        return SketchRule(SketchKind.adaptive_factor_cols, q, ProbabilityRule.uniform, contiguous_partition(n, q))

    @staticmethod
    def adaptive_gauss(q: int) -> "SketchRule":
        return SketchRule(SketchKind.adaptive_factor_gauss, q, ProbabilityRule.none)

    @staticmethod
    def adaptive_gauss_device(q: int) -> "SketchRule":
        return SketchRule(SketchKind.adaptive_factor_gauss_device, q, ProbabilityRule.none)

    @staticmethod
    def adaptive_cols_uniform(q: int) -> "SketchRule":
        """Paper sampler: q distinct coordinates uniformly; not in the reference."""
        return SketchRule(SketchKind.adaptive_factor_cols_uniform, q, ProbabilityRule.uniform)

    def is_adaptive(self) -> bool:
        return self.kind in (SketchKind.adaptive_factor_cols, SketchKind.adaptive_factor_gauss,
                             SketchKind.adaptive_factor_cols_uniform, SketchKind.adaptive_factor_gauss_device)

    def describe(self) -> str:
        return f"{self.kind.name}(q={self.q})"


@dataclass
class TrackOptions:  # simi.hpp:53-57
    residual_every_k: int = 10
    flops: bool = True
    wall_time: bool = True


@dataclass
class HistoryPoint:  # simi.hpp:73-78
    k: int
    residual: float
    flops: float
    seconds: float


@dataclass
class InverterState:  # simi.hpp:82-90
    x: Optional[np.ndarray] = None
    k: int = 0
    history: list = field(default_factory=list)
    max_symmetry_drift: float = 0.0
    flops: float = 0.0
    seconds: float = 0.0
    l: Optional[np.ndarray] = None  # AdaRBFGS factor (FactoredState::l)
    x_inv: Optional[np.ndarray] = None  # dfp's tracked inverse iterate (simi.hpp:86)
    redraws: int = 0


@dataclass
class RunResult:  # simi.hpp:92-96
    state: InverterState
    termination: Termination = Termination.error
    message: str = ""


@dataclass
class InverterConfig:  # simi.hpp:59-71 (named bfgs method)
    a: ProblemMatrix
    rule: SketchRule = field(default_factory=lambda: SketchRule.gaussian(1))
    tol: float = 1e-2
    max_iters: int = 1000
    time_budget_seconds: float = 0.0
    seed: int = 0
    track: TrackOptions = field(default_factory=TrackOptions)
    x0: Optional[np.ndarray] = None
    max_redraws: int = 100
    on_checkpoint: Optional[Callable[[HistoryPoint], None]] = None  # addition
    return_x: bool = True
    update: UpdateName = UpdateName.bfgs  # MethodSpec::named_method(update)


@dataclass
class BaselineConfig:  # baselines.hpp:55-64
    a: ProblemMatrix
    method: BaselineMethod = BaselineMethod.newton_schulz
    tol: float = 1e-2
    max_iters: int = 1000
    time_budget_seconds: float = 0.0
    seed: int = 0  # spectral-norm start vector for the paper init
    track: TrackOptions = field(default_factory=TrackOptions)
    x0: Optional[np.ndarray] = None  # default: the method's paper initialisation
    on_checkpoint: Optional[Callable[[HistoryPoint], None]] = None
    return_x: bool = True


@dataclass
class AdaConfig:  # adarbfgs.hpp:46-56
    a: ProblemMatrix
    rule: SketchRule = field(default_factory=lambda: SketchRule.adaptive_gauss(1))
    tol: float = 1e-2
    max_iters: int = 1000
    time_budget_seconds: float = 0.0
    seed: int = 0
    track: TrackOptions = field(default_factory=TrackOptions)
    l0: Optional[np.ndarray] = None
    max_redraws: int = 100
    on_checkpoint: Optional[Callable[[HistoryPoint], None]] = None
    return_x: bool = True
    return_l: bool = True


def _cfg(rule: SketchRule, tol, max_iters, budget, seed, track, x0, max_redraws, cb):
    c = L.InverterConfigC()
    L.load().si_default_config(C.byref(c))
    c.sketch = int(rule.kind)
    c.probabilities = 1 if rule.probabilities == ProbabilityRule.convenient else 0
    c.q = int(rule.q)
    c.tol = float(tol)
    c.max_iters = int(max_iters)
    c.time_budget_seconds = float(budget)
    c.seed = int(seed) & (2**64 - 1)
    c.residual_every_k = int(track.residual_every_k)
    c.track_flops = 1 if track.flops else 0
    c.track_wall_time = 1 if track.wall_time else 0
    c.max_redraws = int(max_redraws)
    keep = []
    if x0 is not None:
        x0a = _f64(x0)
        keep.append(x0a)
        c.x0_host = _pd(x0a)
    if cb is not None:
        def _tramp(pt, _user):
            hp = C.cast(pt, C.POINTER(L.HistoryPoint)).contents
            cb(HistoryPoint(int(hp.k), float(hp.residual), float(hp.flops), float(hp.seconds)))
        fn = L.CHECKPOINT_FN(_tramp)
        keep.append(fn)
        c.on_checkpoint = fn
    return c, keep


def run_inverter(config: InverterConfig, out: Optional[np.ndarray] = None) -> RunResult:
    """RunResult run_inverter(const InverterConfig&) for MethodSpec::named_method(config.update)
    (simi.cpp:217-381): bfgs, psb, aip or dfp; state.x_inv is dfp's tracked inverse.

    `out` (optional): caller-provided n×n Fortran-ordered float64 buffer for the
    final X (e.g. pinned host memory)."""
    a = config.a
    if config.rule.is_adaptive():
        raise ConfigError("run_inverter: adaptive sketch rules belong to the adarbfgs driver")
    n = a.n()
    if config.x0 is not None and np.shape(config.x0) != (n, n):
        raise ConfigError("run_inverter: x0 dimension mismatch")
    update = UpdateName(config.update)
    c, keep = _cfg(config.rule, config.tol, config.max_iters, config.time_budget_seconds, config.seed, config.track,
                   config.x0, config.max_redraws, config.on_checkpoint)
    c.update = int(update)
    cap = int(config.max_iters) // max(1, config.track.residual_every_k) + 4
    hist = (L.HistoryPoint * cap)()
    res = L.RunResultC()
    if out is not None:
        if out.shape != (n, n) or out.dtype != np.float64 or not out.flags.f_contiguous:
            raise ConfigError("run_inverter: out must be an n×n Fortran-ordered float64 array")
        x = out
    else:
        x = np.empty((n, n), order="F") if config.return_x else None
    xi = np.empty((n, n), order="F") if (update == UpdateName.dfp and config.return_x) else None
    _check(L.load().si_run_inverter_pair(a.ctx.handle, a.handle, C.byref(c), _pd(x) if x is not None else None,
                                         _pd(xi) if xi is not None else None, hist, cap, C.byref(res)))
    del keep
    m = min(int(res.history_count), cap)
    st = InverterState(x=x, k=int(res.k),
                       history=[HistoryPoint(int(h.k), h.residual, h.flops, h.seconds) for h in hist[:m]],
                       max_symmetry_drift=res.max_symmetry_drift, flops=res.flops, seconds=res.seconds,
                       redraws=int(res.redraws), x_inv=xi)
    return RunResult(st, Termination(res.termination), res.message.decode(errors="replace"))


def run_baseline(config: BaselineConfig) -> RunResult:
    """RunResult run_baseline(const BaselineConfig&) (baselines.cpp:52-151): Newton–Schulz
    X⁺ = 2X − XAX or minimal residual with the carried residual, on the GPU."""
    a = config.a
    n = a.n()
    if config.x0 is not None and np.shape(config.x0) != (n, n):
        raise ConfigError("run_baseline: x0 dimension mismatch")
    c, keep = _cfg(SketchRule.gaussian(1), config.tol, config.max_iters, config.time_budget_seconds, config.seed,
                   config.track, config.x0, 0, config.on_checkpoint)
    cap = int(config.max_iters) // max(1, config.track.residual_every_k) + 4
    hist = (L.HistoryPoint * cap)()
    res = L.RunResultC()
    x = np.empty((n, n), order="F") if config.return_x else None
    _check(L.load().si_run_baseline(a.ctx.handle, a.handle, int(BaselineMethod(config.method)), C.byref(c),
                                    _pd(x) if x is not None else None, hist, cap, C.byref(res)))
    del keep
    m = min(int(res.history_count), cap)
    st = InverterState(x=x, k=int(res.k),
                       history=[HistoryPoint(int(h.k), h.residual, h.flops, h.seconds) for h in hist[:m]],
                       flops=res.flops, seconds=res.seconds)
    return RunResult(st, Termination(res.termination), res.message.decode(errors="replace"))


def run_adarbfgs(config: AdaConfig) -> RunResult:
    """RunResult run_adarbfgs(const AdaConfig&) (adarbfgs.cpp:91-200); state.x = L·Lᵀ, state.l = L."""
    a = config.a
    if not config.rule.is_adaptive():
        raise ConfigError("run_adarbfgs: rule must be adaptive")
    n = a.n()
    if config.l0 is not None and np.shape(config.l0) != (n, n):
        raise ConfigError("run_adarbfgs: l0 dimension mismatch")
    c, keep = _cfg(config.rule, config.tol, config.max_iters, config.time_budget_seconds, config.seed, config.track,
                   config.l0, config.max_redraws, config.on_checkpoint)
    cap = int(config.max_iters) // max(1, config.track.residual_every_k) + 4
    hist = (L.HistoryPoint * cap)()
    res = L.RunResultC()
    lo = np.empty((n, n), order="F") if config.return_l else None
    xo = np.empty((n, n), order="F") if config.return_x else None
    _check(L.load().si_run_adarbfgs(a.ctx.handle, a.handle, C.byref(c), _pd(lo) if lo is not None else None,
                                    _pd(xo) if xo is not None else None, hist, cap, C.byref(res)))
    del keep
    m = min(int(res.history_count), cap)
    st = InverterState(x=xo, l=lo, k=int(res.k),
                       history=[HistoryPoint(int(h.k), h.residual, h.flops, h.seconds) for h in hist[:m]],
                       flops=res.flops, seconds=res.seconds, redraws=int(res.redraws))
    return RunResult(st, Termination(res.termination), res.message.decode(errors="replace"))


# ------------------------------------------------------------- step level --


def bfgs_step(x, a, s, *, context: Optional[Context] = None) -> np.ndarray:
    """Matrix bfgs_step(const Matrix& x, const Matrix& a, const Matrix& s) (qn_updates.hpp:70).

    Raises GramRankDeficientError when SᵀAS is not positive definite (the resample signal)."""
    ctx = context or default_context()
    x, a, s = _f64(x), _f64(a), _f64(s)
    n, q = s.shape
    if x.shape != (n, n) or a.shape != (n, n):
        raise ConfigError("bfgs_step: dimension mismatch")
    out = np.empty((n, n), order="F")
    _check(L.load().si_bfgs_step(ctx.handle, n, q, _pd(x), _pd(a), _pd(s), _pd(out)))
    return out


def _named_step(fn, name, x, a, s, context):
    ctx = context or default_context()
    x, a, s = _f64(x), _f64(a), _f64(s)
    n, q = s.shape
    if x.shape != (n, n) or a.shape != (n, n):
        raise ConfigError(f"{name}: dimension mismatch")
    out = np.empty((n, n), order="F")
    _check(fn(ctx.handle, n, q, _pd(x), _pd(a), _pd(s), _pd(out)))
    return out


def psb_step(x, a, s, *, context: Optional[Context] = None) -> np.ndarray:
    """Matrix psb_step(x, a, s) (qn_updates.cpp:121-129) on the GPU."""
    return _named_step(L.load().si_psb_step, "psb_step", x, a, s, context)


def aip_step(x, a, s, *, context: Optional[Context] = None) -> np.ndarray:
    """Matrix aip_step(x, a, s) (qn_updates.cpp:147-152) on the GPU."""
    return _named_step(L.load().si_aip_step, "aip_step", x, a, s, context)


def dfp_step(x, x_inv, a, s, *, context: Optional[Context] = None):
    """IteratePair dfp_step(x, x_inv, a, s) (qn_updates.cpp:154-174) -> (primal, inverse)."""
    ctx = context or default_context()
    x, xi, a, s = _f64(x), _f64(x_inv), _f64(a), _f64(s)
    n, q = s.shape
    if x.shape != (n, n) or xi.shape != (n, n) or a.shape != (n, n):
        raise ConfigError("dfp_step: dimension mismatch")
    out, outi = np.empty((n, n), order="F"), np.empty((n, n), order="F")
    _check(L.load().si_dfp_step(ctx.handle, n, q, _pd(x), _pd(xi), _pd(a), _pd(s), _pd(out), _pd(outi)))
    return out, outi


def newton_schulz_step(x, a, *, context: Optional[Context] = None) -> np.ndarray:
    """Matrix newton_schulz_step(x, a) = 2X − X·A·X (baselines.cpp:12-14) on the GPU."""
    ctx = context or default_context()
    x, a = _f64(x), _f64(a)
    out = np.empty_like(x, order="F")
    _check(L.load().si_newton_schulz_step(ctx.handle, x.shape[0], _pd(x), _pd(a), _pd(out)))
    return out


def newton_schulz_init(a: ProblemMatrix, seed: int = 0) -> np.ndarray:
    """Matrix newton_schulz_init(a, seed) = 0.99·Aᵀ/s² (baselines.cpp:16-20)."""
    out = np.empty((a.n(), a.n()), order="F")
    _check(L.load().si_newton_schulz_init(a.ctx.handle, a.handle, C.c_uint64(seed), _pd(out)))
    return out


def spectral_norm_estimate(a: ProblemMatrix, iters: int = 100, seed: int = 0) -> float:
    """double spectral_norm_estimate(m, iters, seed) (linalg.cpp:106-129), products on the GPU."""
    out = C.c_double()
    _check(L.load().si_spectral_norm_estimate(a.ctx.handle, a.handle, int(iters), C.c_uint64(seed), C.byref(out)))
    return out.value


def mr_step_cached(x, r, a, *, context: Optional[Context] = None):
    """MrStep mr_step_cached(x, r, a) (baselines.cpp:22-37) -> (x, r, alpha, stagnated)."""
    ctx = context or default_context()
    x, r, a = _f64(x), _f64(r), _f64(a)
    n = x.shape[0]
    xo, ro = np.empty((n, n), order="F"), np.empty((n, n), order="F")
    al, stg = C.c_double(), C.c_int()
    _check(L.load().si_mr_step_cached(ctx.handle, n, _pd(x), _pd(r), _pd(a), _pd(xo), _pd(ro), C.byref(al),
                                      C.byref(stg)))
    return xo, ro, al.value, bool(stg.value)


def mr_init(a: ProblemMatrix) -> np.ndarray:
    """Matrix mr_init(a) = Tr(A)/Tr(AAᵀ)·I (baselines.cpp:45-50)."""
    out = np.empty((a.n(), a.n()), order="F")
    _check(L.load().si_mr_init(a.ctx.handle, a.handle, _pd(out)))
    return out


def adarbfgs_update_factor(l, a, stilde, *, context: Optional[Context] = None) -> np.ndarray:
    """Matrix adarbfgs_update_factor(l, a, stilde) (adarbfgs.hpp:28)."""
    ctx = context or default_context()
    l, a, st = _f64(l), _f64(a), _f64(stilde)
    n, q = st.shape
    if l.shape != (n, n) or a.shape != (n, n):
        raise ConfigError("adarbfgs_update_factor: dimension mismatch")
    out = np.empty((n, n), order="F")
    rc = L.load().si_adarbfgs_update_factor(ctx.handle, n, q, _pd(l), _pd(a), _pd(st), _pd(out))
    if rc == 6:  # floor hit: the reference throws NumericalError (linalg.cpp:150-151)
        raise NumericalError(L.load().si_last_error().decode())
    _check(rc)
    return out


def sym_inv_sqrt(m, *, context: Optional[Context] = None) -> np.ndarray:
    """Matrix sym_inv_sqrt(const Matrix& m) (linalg.cpp:144-155) on the GPU: M^{-1/2};
    raises NumericalError iff an eigenvalue λ ≤ 1e-14·λmax or λ ≤ 0."""
    ctx = context or default_context()
    m = _f64(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ConfigError("sym_inv_sqrt: matrix must be square")
    q = m.shape[0]
    out = np.empty((q, q), order="F")
    _check(L.load().si_sym_inv_sqrt(ctx.handle, q, _pd(m), _pd(out)))
    return out


def adaptive_block_probabilities(l, a, blocks: Sequence[Sequence[int]], *, context: Optional[Context] = None):
    """Vector adaptive_block_probabilities(l, a, blocks) (adarbfgs.hpp:32-33)."""
    ctx = context or default_context()
    l, a = _f64(l), _f64(a)
    n = l.shape[0]
    offs = np.zeros(len(blocks) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(b) for b in blocks])
    idx = np.ascontiguousarray(np.concatenate([np.asarray(b, dtype=np.int64) for b in blocks]) if blocks
                               else np.zeros(0, np.int64))
    out = np.empty(len(blocks))
    _check(L.load().si_adaptive_block_probabilities(ctx.handle, n, _pd(l), _pd(a), len(blocks),
                                                    offs.ctypes.data_as(L.pi64), idx.ctypes.data_as(L.pi64),
                                                    _pd(out)))
    return out


def residual(a: ProblemMatrix, x) -> float:
    """‖I − A X‖_F on the device (simi.cpp:242-244)."""
    x = _f64(x)
    out = C.c_double()
    _check(L.load().si_residual(a.ctx.handle, a.handle, _pd(x), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- flops ----


def flops_bfgs(n, q) -> float:  # flops.cpp:43-46
    n, q = float(n), float(q)
    return 10 * n * n * q + 10 * n * q * q + 2 * q ** 3 + 4 * n * n


def flops_adarbfgs(n, q) -> float:  # flops.cpp:70-74
    n, q = float(n), float(q)
    return 8 * n * n * q + 10 * n * q * q + 4 * q ** 3 + n * q + n * n


# ------------------------------------------------------------------ RNG ----


class RngStream:
    """The reference's RngStream (rng.hpp:13-71), host side of the product library."""

    def __init__(self, seed: int = 0, _handle=None):
        lib = L.load()
        if _handle is None:
            h = C.c_void_p()
            _check(lib.si_rng_create(C.c_uint64(seed & (2**64 - 1)), C.byref(h)))
            _handle = h
        self._h = _handle

    def substream(self, index: int) -> "RngStream":
        h = C.c_void_p()
        _check(L.load().si_rng_substream(self._h, C.c_uint64(index), C.byref(h)))
        return RngStream(_handle=h)

    def uniform(self) -> float:
        return float(L.load().si_rng_uniform(self._h))

    def gaussian(self) -> float:
        return float(L.load().si_rng_gaussian(self._h))

    def categorical(self, p) -> int:
        p = np.ascontiguousarray(p, dtype=np.float64)
        return int(L.load().si_rng_categorical(self._h, _pd(p), p.size))

    def uniform_index(self, n: int) -> int:
        return int(L.load().si_rng_uniform_index(self._h, n))

    def gaussian_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), order="F")
        _check(L.load().si_rng_gaussian_matrix(self._h, rows, cols, _pd(out)))
        return out

    def uniform_matrix(self, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), order="F")
        _check(L.load().si_rng_uniform_matrix(self._h, rows, cols, _pd(out)))
        return out

    def uniform_subset(self, n: int, q: int) -> np.ndarray:
        out = np.empty(q, dtype=np.int64)
        _check(L.load().si_rng_uniform_subset(self._h, n, q, out.ctypes.data_as(L.pi64)))
        return out

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                L.load().si_rng_destroy(self._h)
                self._h = None
        except Exception:
            pass


# --------------------------------------------------------------- solver ----


@dataclass
class FactoredState:  # adarbfgs.hpp:15-22 (the step-level subset)
    l: np.ndarray
    k: int = 0


def adarbfgs_step(state: FactoredState, a: ProblemMatrix, rule: SketchRule, rng: RngStream,
                  max_redraws: int = 100) -> FactoredState:
    """FactoredState adarbfgs_step(state, a, rule, rng, max_redraws) (adarbfgs.cpp:49-75):
    one factored update on the GPU, drawing from the caller's RngStream."""
    if not rule.is_adaptive() or rule.kind == SketchKind.adaptive_factor_gauss_device:
        raise ConfigError("adarbfgs_step: rule must be adaptive-factor-cols or -gauss")
    n = a.n()
    l = _f64(state.l)
    if l.shape != (n, n):
        raise ConfigError("adarbfgs_step: state dimension mismatch")
    out = np.empty((n, n), order="F")
    _check(L.load().si_adarbfgs_step(a.ctx.handle, a.handle, int(rule.kind), int(rule.q), rng._h, int(max_redraws),
                                     _pd(l), _pd(out)))
    return FactoredState(out, state.k + 1)


class Method(enum.IntEnum):
    rbfgs = 0
    adarbfgs = 1


class Solver:
    """Device-resident iterate (X for RBFGS, L for AdaRBFGS) for benchmarking
    and the row-sharded multi-GPU driver; iterations run without host round trips."""

    def __init__(self, a: ProblemMatrix, method: Method, rule: SketchRule, seed: int = 0):
        self.a = a
        self.ctx = a.ctx
        self.q = rule.q
        h = C.c_void_p()
        _check(L.load().si_solver_create(self.ctx.handle, a.handle, int(method), int(rule.kind), int(rule.q),
                                         C.c_uint64(seed & (2**64 - 1)), C.byref(h)))
        self._h = h

    def set_identity(self):
        _check(L.load().si_solver_set_identity(self._h))

    def set_iterate(self, m):
        m = _f64(m)
        _check(L.load().si_solver_set_iterate(self._h, _pd(m)))

    def iterate(self) -> np.ndarray:
        n = self.a.n()
        out = np.empty((n, n), order="F")
        _check(L.load().si_solver_get_iterate(self._h, _pd(out)))
        return out

    def iterate_device_ptr(self) -> int:
        return int(L.load().si_solver_iterate_device(self._h))

    def step(self, iters: int = 1):
        _check(L.load().si_solver_step(self._h, int(iters)))

    def step_with_sketch(self, s=None, idx=None):
        sp = None
        ip = None
        if s is not None:
            s = _f64(s)
            sp = _pd(s)
        if idx is not None:
            idx = np.ascontiguousarray(idx, dtype=np.int64)
            ip = idx.ctypes.data_as(L.pi64)
        _check(L.load().si_solver_step_with_sketch(self._h, sp, ip))

    def residual(self) -> float:
        out = C.c_double()
        _check(L.load().si_solver_residual(self._h, C.byref(out)))
        return out.value

    def redraws(self) -> int:
        return int(L.load().si_solver_redraws(self._h))

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                L.load().si_solver_destroy(self._h)
                self._h = None
        except Exception:
            pass
