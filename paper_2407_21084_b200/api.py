"""Python mirror of the reference's Python surface for the backward-solve path.

The reference exposes ``qrmc.solve(bench, gamma, measure, steps, paths,
damping, seed, workers, memory_mode)`` returning a ``CoefficientTable``
(proj/bindings/py_core.cpp:172-187; classes at py_core.cpp:41-170). This
module keeps those names, argument meanings and error types, and routes the
solve through the C ABI of ``_lib/libqrmc_gpu.so`` (include/qrmc_gpu.h) on a
B200. Exceptions follow the reference's taxonomy (errors.hpp): ValueError for
std::invalid_argument, NumericError, SimulationError(step), CapacityError.
There is no CPU fallback: without the CUDA library every solve raises.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi


class QrmcError(RuntimeError):
    pass


class CapacityError(QrmcError):
    """qrmc::CapacityError (errors.hpp:9-13)."""


class SimulationError(QrmcError):
    """qrmc::SimulationError (errors.hpp:15-25); ``step`` as in the reference."""

    def __init__(self, msg: str, step: int):
        super().__init__(msg)
        self.step = step


class NumericError(QrmcError):
    """qrmc::NumericError (errors.hpp:27-31)."""


class DeviceError(QrmcError):
    """CUDA / NCCL failure (no reference analogue)."""


def raise_for(status: int, msg: str, step: int = -1) -> None:
    if status == _abi.OK:
        return
    if status == _abi.EINVAL:
        raise ValueError(msg)
    if status == _abi.ECAPACITY:
        raise CapacityError(msg)
    if status == _abi.ESIM:
        raise SimulationError(msg, step)
    if status == _abi.ENUMERIC:
        raise NumericError(msg)
    if status == _abi.ELOGIC:
        raise IndexError(msg)
    if status == _abi.ENOTIMPL:
        raise NotImplementedError(msg)
    raise DeviceError(f"{_abi.STATUS_NAMES.get(status, status)}: {msg}")


def _err():
    return C.create_string_buffer(1024)


# ---------------------------------------------------------------- plugin surface
@dataclass(frozen=True)
class Measure:
    """SamplingMeasure (proj/include/qrmc/student.hpp:23-61): any mu > 0 on the device (mu = 1, 2
    closed forms; general mu through include/qrmc_student_t.h)."""

    mu: float
    dim: int
    center: tuple = ()

    def __post_init__(self):
        if not (self.mu > 0.0) or not math.isfinite(self.mu):
            raise ValueError("SamplingMeasure: mu must be positive and finite")
        if self.dim < 1:
            raise ValueError("SamplingMeasure: dim must be >= 1")
        if self.center and len(self.center) != self.dim:
            raise ValueError("SamplingMeasure: center size must equal dim")


@dataclass(frozen=True)
class MultiIndexSet:
    """MultiIndexSet descriptor (proj/include/qrmc/multi_index.hpp:23-63).
    Enumeration happens in the C library, bit-exact in order with the reference."""

    kind: str
    dim: int
    degrees: tuple

    @staticmethod
    def full(degrees) -> "MultiIndexSet":
        return MultiIndexSet("full", len(degrees), tuple(int(d) for d in degrees))

    @staticmethod
    def total(dim: int, degree: int) -> "MultiIndexSet":
        return MultiIndexSet("total", dim, (int(degree),))

    @staticmethod
    def hyperbolic(dim: int, degree: int) -> "MultiIndexSet":
        return MultiIndexSet("hyperbolic", dim, (int(degree),))

    @property
    def kind_id(self) -> int:
        return _abi.GAMMA_KINDS[self.kind]

    def __len__(self) -> int:
        L = _abi.lib()
        deg = (C.c_int32 * len(self.degrees))(*self.degrees)
        n = L.qrmc_gpu_gamma_size(self.kind_id, self.dim, deg, len(self.degrees))
        if n < 0:
            raise_for(int(-n), "multi-index set construction failed")
        return int(n)

    def indices(self) -> np.ndarray:
        n = len(self)
        out = np.zeros((n, self.dim), dtype=np.int32)
        deg = (C.c_int32 * len(self.degrees))(*self.degrees)
        err = _err()
        st = _abi.lib().qrmc_gpu_gamma_indices(self.kind_id, self.dim, deg, len(self.degrees),
                                               out.ctypes.data_as(C.POINTER(C.c_int32)), out.size,
                                               err, 1024)
        raise_for(st, err.value.decode())
        return out


@dataclass(frozen=True)
class SinBenchmark:
    """SinBenchmark (proj/include/qrmc/benchmark.hpp:18-26)."""

    dim: int
    kappa: float = 0.6
    lambda_: float = 0.0
    horizon: float = 1.0

    @property
    def lam(self) -> float:
        return self.lambda_ if self.lambda_ > 0.0 else 1.0 / math.sqrt(float(self.dim))

    def problem(self) -> _abi.Problem:
        return _abi.sin_bench_problem(self.dim, self.kappa, self.lambda_, self.horizon)


def exact_solution(t: float, x, bench: SinBenchmark) -> float:
    """Closed form u(t, x) of the benchmark (benchmark.cpp:20-28)."""
    s = 0.0
    for v in np.asarray(x, dtype=np.float64).ravel():
        s += float(v)
    lam = bench.lam
    return 1.0 + bench.kappa + math.sin(lam * s) * math.exp(lam * lam * bench.dim * (t - bench.horizon) / 2.0)


@dataclass
class TruncationStats:
    applications: int = 0
    clipped: int = 0

    def clip_fraction(self) -> float:
        return 0.0 if self.applications == 0 else self.clipped / self.applications


def make_config(steps, paths, damping, seed, workers, memory_mode, gamma: MultiIndexSet,
                measure: Measure) -> _abi.ConfigHolder:
    mode = {"store": _abi.MEMORY_STORE, "store_cloud": _abi.MEMORY_STORE,
            "recompute": _abi.MEMORY_RECOMPUTE, "recompute_from_seeds": _abi.MEMORY_RECOMPUTE}
    if memory_mode not in mode:
        raise ValueError(f"unknown memory mode: {memory_mode}")
    if gamma.dim != measure.dim:
        raise ValueError("RunConfig: gamma/measure dims must equal spec.dim")
    return _abi.ConfigHolder(steps=steps, paths=paths, damping=damping, seed=seed, workers=workers,
                             memory_mode=mode[memory_mode], gamma_kind=gamma.kind_id,
                             degrees=gamma.degrees, mu=measure.mu,
                             center=list(measure.center) if measure.center else None)


@dataclass
class CoefficientTable:
    """CoefficientTable (proj/include/qrmc/solver.hpp:51-67)."""

    steps: int
    paths: int
    damping: float
    seed: int
    horizon: float
    measure: Measure
    gamma: MultiIndexSet
    table: np.ndarray  # [steps][basis_size]
    truncation: TruncationStats = field(default_factory=TruncationStats)
    step_wall_seconds: np.ndarray | None = None
    device_seconds: float = 0.0
    kernel_launches: int = 0

    def dt(self) -> float:
        return self.horizon / self.steps

    def coefficients(self, i: int) -> np.ndarray:
        if not (0 <= i < self.steps):
            raise IndexError("step not computed")
        return self.table[i].copy()

    def _config(self) -> _abi.ConfigHolder:
        return make_config(self.steps, self.paths, self.damping, self.seed, 0, "store", self.gamma,
                           self.measure)

    def evaluate(self, i: int, x) -> float | np.ndarray:
        """evaluate_solution(table, i, x) (solver.cpp:228-237), on the device."""
        if not (0 <= i < self.steps):
            raise IndexError("evaluate_solution: step index out of range")
        pts = np.ascontiguousarray(x, dtype=np.float64)
        scalar = pts.ndim == 1
        pts = pts.reshape(-1, self.gamma.dim)
        out = np.zeros(pts.shape[0])
        cfg = self._config()
        row = np.ascontiguousarray(self.table[i])
        err = _err()
        st = _abi.lib().qrmc_gpu_evaluate(cfg.ref(), self.gamma.dim,
                                          row.ctypes.data_as(C.POINTER(C.c_double)),
                                          pts.ctypes.data_as(C.POINTER(C.c_double)), pts.shape[0],
                                          out.ctypes.data_as(C.POINTER(C.c_double)), err, 1024)
        raise_for(st, err.value.decode())
        return float(out[0]) if scalar else out

    # ---- artifacts (proj/src/table_io.cpp) ----
    def to_json(self) -> str:
        """table_to_json (table_io.cpp:45-73): the `qrmc.coefficients.v1` document,
        byte-identical to the reference's for the same table."""
        cfg = self._config()
        coeffs = np.ascontiguousarray(self.table, dtype=np.float64)
        err = _err()
        L = _abi.lib()
        args = (cfg.ref(), self.gamma.dim, float(self.horizon), coeffs.ctypes.data_as(C.POINTER(C.c_double)))
        n = L.qrmc_gpu_table_json(*args, None, 0, err, 1024)
        if n < 0:
            raise_for(int(-n), err.value.decode())
        buf = C.create_string_buffer(int(n))
        n = L.qrmc_gpu_table_json(*args, buf, int(n), err, 1024)
        if n < 0:
            raise_for(int(-n), err.value.decode())
        return buf.value.decode()

    def save_json(self, path) -> None:
        """save_table_json (table_io.cpp:75-81): the document plus a newline."""
        with open(path, "wb") as f:
            f.write(self.to_json().encode() + b"\n")

    @staticmethod
    def from_json(text: str) -> "CoefficientTable":
        """table_from_json (table_io.cpp:83-125): schema, step range, entry count and
        index order are checked; IoError cases raise ValueError."""
        import json

        try:
            doc = json.loads(text)
        except ValueError as e:
            raise ValueError(f"coefficient artifact: parse error: {e}") from e
        try:
            if doc["schema"] != "qrmc.coefficients.v1":
                raise ValueError("coefficient artifact: unknown schema")
            cfg = doc["config"]
            m, g = cfg["measure"], cfg["gamma"]
            measure = Measure(float(m["mu"]), int(m["dim"]), tuple(float(c) for c in m["center"]))
            kind, dim, degrees = g["kind"], int(g["dim"]), tuple(int(v) for v in g["degrees"])
            if kind == "full":
                gamma = MultiIndexSet.full(degrees)
            else:
                if len(degrees) != 1:
                    raise ValueError("gamma descriptor: total/hyperbolic take one degree")
                gamma = MultiIndexSet(kind, dim, degrees)
            rows = gamma.indices()
            steps = int(cfg["steps"])
            table = np.zeros((steps, rows.shape[0]))
            for st in doc["coefficients"]:
                i = int(st["step"])
                if not (0 <= i < steps):
                    raise ValueError("coefficient artifact: step index out of range")
                entries = st["entries"]
                if len(entries) != rows.shape[0]:
                    raise ValueError("coefficient artifact: entry count != basis size")
                for k, (idx, v) in enumerate(entries):
                    if tuple(idx) != tuple(rows[k]):
                        raise ValueError("coefficient artifact: index order mismatch")
                    table[i, k] = float(v)
            return CoefficientTable(steps, int(cfg["paths"]), float(cfg["damping"]), int(cfg["seed"]),
                                    float(cfg["horizon"]), measure, gamma, table)
        except (KeyError, TypeError) as e:
            raise ValueError(f"coefficient artifact: malformed document: {e}") from e

    @staticmethod
    def load_json(path) -> "CoefficientTable":
        with open(path, "rb") as f:
            return CoefficientTable.from_json(f.read().decode())


def backward_solve(problem: _abi.Problem, config: _abi.ConfigHolder, session=None):
    """qrmc::backward_solve (solver.hpp:91) through the C ABI.
    Returns (coefficients [N][K], Stats, step_wall_seconds)."""
    L = _abi.lib()
    deg = config.c.degrees
    K = L.qrmc_gpu_gamma_size(config.c.gamma_kind, problem.dim, deg, config.c.n_degrees)
    if K < 0:
        raise_for(int(-K), "multi-index set construction failed")
    steps = max(int(config.c.steps), 0)
    coeffs = np.zeros((steps, int(K)))
    wall = np.zeros(max(steps, 1))
    stats = _abi.Stats()
    err = _err()
    st = L.qrmc_gpu_backward_solve(session, C.byref(problem), config.ref(),
                                   coeffs.ctypes.data_as(C.POINTER(C.c_double)), coeffs.size,
                                   wall.ctypes.data_as(C.POINTER(C.c_double)), C.byref(stats),
                                   err, 1024)
    raise_for(st, err.value.decode(), stats.error_step)
    return coeffs, stats, wall[:steps]


def solve(bench: SinBenchmark, gamma: MultiIndexSet, measure: Measure, steps: int, paths: int,
          damping: float = 0.0, seed: int = 0, workers: int = 0,
          memory_mode: str = "store") -> CoefficientTable:
    """``qrmc.solve`` (py_core.cpp:172-187): backward-solve the benchmark problem."""
    cfg = make_config(steps, paths, damping, seed, workers, memory_mode, gamma, measure)
    coeffs, stats, wall = backward_solve(bench.problem(), cfg)
    return CoefficientTable(steps=steps, paths=paths, damping=damping, seed=seed,
                            horizon=bench.horizon, measure=measure, gamma=gamma, table=coeffs,
                            truncation=TruncationStats(int(stats.applications), int(stats.clipped)),
                            step_wall_seconds=wall, device_seconds=float(stats.device_seconds),
                            kernel_launches=int(stats.kernel_launches))


@dataclass
class MetricReport:
    mse_max: float
    mse_av: float
    mse_max_undamped: float
    mse_av_undamped: float
    eval_points_per_step: int
    step_squared_error: np.ndarray
    stat_error_indicator: float = 0.0


def mse_metrics(table: CoefficientTable, bench: SinBenchmark, eval_seed: int,
                eval_points: int = 1000, workers: int = 0) -> MetricReport:
    """``qrmc.mse_metrics`` (benchmark.cpp:86-151), evaluated on the device."""
    if table.gamma.dim != bench.dim:
        raise ValueError("mse_metrics: table/benchmark dims differ")
    cfg = table._config()
    out = np.zeros(6)
    step_sq = np.zeros(table.steps)
    coeffs = np.ascontiguousarray(table.table)
    err = _err()
    st = _abi.lib().qrmc_gpu_mse_metrics(cfg.ref(), bench.dim, bench.kappa, bench.lambda_,
                                         bench.horizon, coeffs.ctypes.data_as(C.POINTER(C.c_double)),
                                         eval_seed, eval_points,
                                         out.ctypes.data_as(C.POINTER(C.c_double)),
                                         step_sq.ctypes.data_as(C.POINTER(C.c_double)), err, 1024)
    raise_for(st, err.value.decode())
    return MetricReport(out[0], out[1], out[2], out[3], eval_points, step_sq)


def confidence_interval(values, level: float = 0.99):
    """Normal-approximation CI (benchmark.cpp:153-169)."""
    from statistics import NormalDist

    v = [float(x) for x in values]
    if len(v) < 2:
        raise ValueError("confidence_interval: need at least 2 values")
    if not (0.0 < level < 1.0):
        raise ValueError("confidence_interval: level must be in (0,1)")
    n = float(len(v))
    mean = sum(v) / n
    sd = math.sqrt(sum((x - mean) ** 2 for x in v) / (n - 1.0))
    z = NormalDist().inv_cdf((1.0 + level) / 2.0)
    half = z * sd / math.sqrt(n)
    return mean - half, mean + half
