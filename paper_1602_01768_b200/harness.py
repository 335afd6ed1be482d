"""Benchmark harness with the reference's trace wire format.

Mirrors proj/include/stochinv/bench.hpp:13-68 and proj/src/bench.cpp:16-280 for
the methods that run on the B200 path:

    MatrixSource      mtx / libsvm / synthetic / identity   (bench.cpp:17-27)
    MethodConfig      name, q (0 = ceil(sqrt(n))), probabilities
    BenchmarkSpec     tol, max_iters, time budget, seed, trials, init, residual_every_k,
                      measure_time (False -> byte-identical CSVs across runs)
    run_benchmark     one trace per (method, trial) in method order, trial order;
                      per-trial seed = spec.seed ^ (0x9e3779b97f4a7c15·(4096·i + t + 1))
                      (bench.cpp:122-126); a failing trial records status "error"
                      and the single point {0, 1, 0, 0} (bench.cpp:131-136)
    write_csv         "method,iter,residual,flops,seconds", %.17g through the C
                      library's snprintf (the reference's fmt, bench.cpp:167-172),
                      "#trial" suffix when any trial > 0 (bench.cpp:174-189)
    write_svg         residual-vs-seconds and residual-vs-flops panels, log y

Methods on the GPU path: bfgs (coordinate / coordinate-block sketches, as the
reference's bench drives it, bench.cpp:92-99), psb, aip, dfp (row f3),
adarbfgs-cols, adarbfgs-gauss, newton-schulz, mr (row f4).  The reference's
other update families (row/col/sym/kaczmarz/bad-broyden/good-broyden/column)
are outside the hot path and raise ConfigError.  Trials run one
after another on the GPU (the reference fans them out over host threads); the
output order is the same.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import api
from .api import ConfigError, HistoryPoint, ProbabilityRule, ProblemMatrix, SketchRule, Symmetry, TrackOptions

_libc = ctypes.CDLL(ctypes.util.find_library("c"))
_libc.snprintf.restype = ctypes.c_int


def fmt(v: float) -> str:
    """%.17g exactly as the reference prints it (glibc snprintf)."""
    buf = ctypes.create_string_buffer(64)
    _libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(float(v)))
    return buf.value.decode()


class MatrixSourceKind(enum.Enum):
    mtx = "mtx"
    libsvm = "libsvm"
    synthetic = "synthetic"
    identity = "identity"


@dataclass
class MatrixSource:  # bench.hpp:15-24
    kind: MatrixSourceKind = MatrixSourceKind.synthetic
    path: str = ""
    lam: float = 1.0  # libsvm ridge parameter
    n: int = 0        # synthetic / identity
    seed: int = 0

    def load(self, context: Optional[api.Context] = None) -> ProblemMatrix:
        if self.kind == MatrixSourceKind.mtx:
            return api.load_matrix_market(self.path, context=context)
        if self.kind == MatrixSourceKind.libsvm:
            return api.build_ridge_hessian(self.path, self.lam, context=context)
        if self.kind == MatrixSourceKind.synthetic:
            return api.gen_synthetic(self.n, self.seed, context=context)
        if self.n < 1:
            raise ConfigError("identity source: n must be >= 1")
        return ProblemMatrix(np.eye(self.n), Symmetry.spd, context=context)

    def describe(self) -> str:
        if self.kind == MatrixSourceKind.mtx:
            return f"mtx({self.path})"
        if self.kind == MatrixSourceKind.libsvm:
            return f"libsvm({self.path}, lambda={self.lam:g})"
        if self.kind == MatrixSourceKind.synthetic:
            return f"synthetic({self.n}, seed={self.seed})"
        return f"identity({self.n})"


@dataclass
class MethodConfig:  # bench.hpp:28-34 (the weight spec of the generic variants is not on this path)
    name: str
    q: int = 0  # 0 = ceil(sqrt(n))
    probabilities: ProbabilityRule = ProbabilityRule.uniform


class InitPolicy(enum.Enum):  # bench.hpp:36-39
    paper = "paper"
    identity = "identity"


@dataclass
class BenchmarkSpec:  # bench.hpp:41-50
    methods: List[MethodConfig] = field(default_factory=list)
    tol: float = 1e-2
    max_iters: int = 1000
    time_budget_seconds: float = 0.0
    seed: int = 0
    trials: int = 1
    init: InitPolicy = InitPolicy.paper
    residual_every_k: int = 10
    measure_time: bool = True


@dataclass
class ConvergenceTrace:  # bench.hpp:52-57
    method: str
    trial: int = 0
    points: List[HistoryPoint] = field(default_factory=list)
    status: str = ""


GPU_METHODS = ("bfgs", "psb", "aip", "dfp", "adarbfgs-cols", "adarbfgs-gauss", "newton-schulz", "mr")
REFERENCE_ONLY = ("row", "col", "sym", "kaczmarz", "bad-broyden", "good-broyden", "column")


def default_q(n: int) -> int:  # bench.cpp:42-44
    return max(1, int(math.ceil(math.sqrt(float(n)))))


def trial_seed(spec_seed: int, method_index: int, trial: int) -> int:  # bench.cpp:122-126
    mult = (0x9E3779B97F4A7C15 * (method_index * 4096 + trial + 1)) & 0xFFFFFFFFFFFFFFFF
    return (spec_seed ^ mult) & 0xFFFFFFFFFFFFFFFF


def _run_method(a: ProblemMatrix, m: MethodConfig, spec: BenchmarkSpec, seed: int) -> api.RunResult:
    n = a.n()
    q = m.q if m.q > 0 else default_q(n)
    track = TrackOptions(residual_every_k=spec.residual_every_k, wall_time=spec.measure_time)
    common = dict(tol=spec.tol, max_iters=spec.max_iters, time_budget_seconds=spec.time_budget_seconds, seed=seed,
                  track=track)
    if m.name in ("newton-schulz", "mr"):
        x0 = np.eye(n) if spec.init == InitPolicy.identity else None
        method = api.BaselineMethod.minimal_residual if m.name == "mr" else api.BaselineMethod.newton_schulz
        return api.run_baseline(api.BaselineConfig(a, method=method, x0=x0, return_x=False, **common))
    if m.name in ("adarbfgs-cols", "adarbfgs-gauss"):
        rule = SketchRule.adaptive_cols(n, q) if m.name == "adarbfgs-cols" else SketchRule.adaptive_gauss(q)
        return api.run_adarbfgs(api.AdaConfig(a, rule, return_x=False, return_l=False, **common))
    # named rank-q updates on coordinate sketches (bench.cpp:92-99): q == 1 -> single coordinates,
    # which draw exactly like blocks of width one
    rule = SketchRule.coordinate_block(n, q, m.probabilities)
    return api.run_inverter(api.InverterConfig(a, rule, update=api.UpdateName(m.name), return_x=False, **common))


def _status(r: api.RunResult) -> str:  # bench.cpp:105-114
    if r.termination == api.Termination.tol_reached:
        return "tol_reached"
    if r.termination == api.Termination.max_iters:
        return "max_iters"
    return "diverged" if r.message.startswith("diverged") else "error"


def run_benchmark(a: ProblemMatrix, spec: BenchmarkSpec) -> List[ConvergenceTrace]:
    """std::vector<ConvergenceTrace> run_benchmark(a, spec) (bench.cpp:141-163)."""
    if not spec.methods:
        raise ConfigError("run_benchmark: at least one method required")
    if spec.tol < 0.0:
        raise ConfigError("run_benchmark: tol must be >= 0")
    if spec.trials < 1:
        raise ConfigError("run_benchmark: trials must be >= 1")
    for m in spec.methods:
        if m.name in REFERENCE_ONLY:
            raise ConfigError(f"run_benchmark: method '{m.name}' is not on the B200 path (SURVEY §8)")
        if m.name not in GPU_METHODS:
            raise ConfigError(f"unknown update name: {m.name}")
    traces = []
    for mi, m in enumerate(spec.methods):
        for t in range(spec.trials):
            tr = ConvergenceTrace(m.name, t)
            try:
                r = _run_method(a, m, spec, trial_seed(spec.seed, mi, t))
                tr.points = list(r.state.history)
                tr.status = _status(r)
            except Exception:  # noqa: BLE001 — the reference records any failure as status "error"
                tr.status = "error"
                tr.points = [HistoryPoint(0, 1.0, 0.0, 0.0)]
            traces.append(tr)
    return traces


def write_csv(traces: List[ConvergenceTrace], path: str) -> None:
    """CSV with header method,iter,residual,flops,seconds; %.17g numbers; "#trial"
    suffix on every label when any trace has trial > 0 (bench.cpp:174-189)."""
    multi = any(t.trial > 0 for t in traces)
    lines = ["method,iter,residual,flops,seconds\n"]
    for t in traces:
        label = f"{t.method}#{t.trial}" if multi else t.method
        for p in t.points:
            lines.append(f"{label},{int(p.k)},{fmt(p.residual)},{fmt(p.flops)},{fmt(p.seconds)}\n")
    try:
        with open(path, "w", newline="\n") as f:
            f.writelines(lines)
    except OSError as e:
        raise api.IoError(f"cannot write {path}") from e


_PALETTE = ("#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b", "#17becf", "#7f7f7f")


def _panel(out: list, traces, x0, y0, w, h, use_seconds: bool, title: str) -> None:
    xs = [p.seconds if use_seconds else p.flops for t in traces for p in t.points]
    xmax = max([v for v in xs] + [0.0]) or 1.0
    pos = [p.residual for t in traces for p in t.points if p.residual > 0.0]
    floor_res = 1e-16
    ymin = max(min(pos + [1.0]) / 2.0, floor_res)
    ymax = max(max([p.residual for t in traces for p in t.points] + [1.0]) * 2.0, ymin * 10.0)
    ly0, ly1 = math.log10(ymin), math.log10(ymax)

    def sx(v):
        return x0 + w * (v / xmax)

    def sy(r):
        return y0 + h * (1.0 - (math.log10(max(r, floor_res)) - ly0) / (ly1 - ly0))

    out.append(f"<rect x='{x0:g}' y='{y0:g}' width='{w:g}' height='{h:g}' fill='none' stroke='black'/>\n")
    out.append(f"<text x='{x0 + w / 2:g}' y='{y0 - 10:g}' text-anchor='middle' font-size='14'>{title}</text>\n")
    for d in range(math.ceil(ly0), math.floor(ly1) + 1):
        y = sy(10.0 ** d)
        out.append(f"<line x1='{x0:g}' y1='{y:g}' x2='{x0 + w:g}' y2='{y:g}' stroke='#dddddd'/>\n")
        out.append(f"<text x='{x0 - 6:g}' y='{y + 4:g}' text-anchor='end' font-size='10'>1e{d}</text>\n")
    unit = " s" if use_seconds else " flops"
    out.append(f"<text x='{x0 + w:g}' y='{y0 + h + 16:g}' text-anchor='end' font-size='10'>{fmt(xmax)}{unit}</text>\n")
    for i, t in enumerate([t for t in traces if t.points]):
        pts = " ".join(f"{sx(p.seconds if use_seconds else p.flops):g},{sy(p.residual):g}" for p in t.points)
        out.append(f"<polyline fill='none' stroke='{_PALETTE[i % 8]}' points='{pts} '/>\n")


def write_svg(traces: List[ConvergenceTrace], path: str) -> None:
    """Self-contained SVG: relative residual vs seconds and vs flops, log-scale y
    (bench.hpp:66-68; the same 980×520 two-panel layout and legend)."""
    out = ["<svg xmlns='http://www.w3.org/2000/svg' version='1.1' width='980' height='520' "
           "viewBox='0 0 980 520'>\n", "<rect width='980' height='520' fill='white'/>\n"]
    _panel(out, traces, 60, 40, 400, 400, True, "relative residual vs seconds")
    _panel(out, traces, 540, 40, 400, 400, False, "relative residual vs flops")
    x, y = 60.0, 475.0
    for i, t in enumerate(traces):
        label = t.method + (f"#{t.trial}" if t.trial > 0 else "") + f" [{t.status}]"
        out.append(f"<rect x='{x:g}' y='{y - 9:g}' width='12' height='12' fill='{_PALETTE[i % 8]}'/>\n")
        out.append(f"<text x='{x + 16:g}' y='{y + 2:g}' font-size='11'>{label}</text>\n")
        x += 180.0
        if x > 900.0:
            x, y = 60.0, y + 18.0
    out.append("</svg>\n")
    try:
        with open(path, "w", newline="\n") as f:
            f.writelines(out)
    except OSError as e:
        raise api.IoError(f"cannot write {path}") from e
