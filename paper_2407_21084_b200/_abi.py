"""ctypes mirror of include/qrmc_gpu.h (the C ABI of the B200 solver).

The structs here are byte-for-byte the C structs; the library itself is
loaded lazily by :func:`lib` and a missing library is an error, never a
fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["QRMC_GPU_LIB"]) if os.environ.get("QRMC_GPU_LIB") else PKG_DIR / "_lib" / "libqrmc_gpu.so"

# qrmc_status
OK, EINVAL, ENUMERIC, ESIM, ECAPACITY, ECUDA, ENCCL, ENOTIMPL, ELOGIC = range(9)
STATUS_NAMES = {
    OK: "OK", EINVAL: "EINVAL", ENUMERIC: "ENUMERIC", ESIM: "ESIM", ECAPACITY: "ECAPACITY",
    ECUDA: "ECUDA", ENCCL: "ENCCL", ENOTIMPL: "ENOTIMPL", ELOGIC: "ELOGIC",
}

GAMMA_FULL, GAMMA_TOTAL, GAMMA_HYPERBOLIC = 0, 1, 2
GAMMA_KINDS = {"full": GAMMA_FULL, "total": GAMMA_TOTAL, "hyperbolic": GAMMA_HYPERBOLIC}
MEMORY_STORE, MEMORY_RECOMPUTE = 0, 1
TERMINAL_SIN_SUM, TERMINAL_CONST, TERMINAL_X0, TERMINAL_NAN = 0, 1, 2, 3
DRIVER_ZERO, DRIVER_CONST, DRIVER_Y, DRIVER_SIN_BENCH = 0, 1, 2, 3
DRIFT_ZERO, DRIFT_CONST, DRIFT_AFFINE = 0, 1, 2
DIFFUSION_IDENTITY, DIFFUSION_SCALAR, DIFFUSION_DIAG = 0, 1, 2


class Problem(C.Structure):
    """qrmc_problem_t -- ProblemSpec (proj/include/qrmc/sde.hpp:18-49)."""

    _fields_ = [
        ("dim", C.c_int32), ("brownian_dim", C.c_int32), ("horizon", C.c_double),
        ("terminal_kind", C.c_int32), ("driver_kind", C.c_int32),
        ("drift_kind", C.c_int32), ("diffusion_kind", C.c_int32),
        ("terminal_params", C.c_double * 4), ("driver_params", C.c_double * 4),
        ("drift_params", C.c_double * 2), ("diffusion_params", C.c_double * 2),
        ("growth_g", C.c_double), ("growth_exp_g", C.c_double), ("growth_f", C.c_double),
        ("growth_exp_f", C.c_double), ("lipschitz_f", C.c_double),
        ("moment_ratio", C.c_double), ("state_bound", C.c_double),
        ("drift_vec", C.c_double * 16), ("diffusion_vec", C.c_double * 8),
    ]


class Config(C.Structure):
    """qrmc_config_t -- RunConfig (proj/include/qrmc/solver.hpp:24-35)."""

    _fields_ = [
        ("steps", C.c_int32), ("workers", C.c_int32), ("paths", C.c_int64),
        ("damping", C.c_double), ("seed", C.c_uint64), ("memory_mode", C.c_int32),
        ("gamma_kind", C.c_int32), ("degrees", C.POINTER(C.c_int32)),
        ("n_degrees", C.c_int32), ("reserved", C.c_int32), ("mu", C.c_double),
        ("center", C.POINTER(C.c_double)),
    ]


class Stats(C.Structure):
    """qrmc_stats_t -- TruncationStats (+ error step, launches, device time)."""

    _fields_ = [
        ("applications", C.c_uint64), ("clipped", C.c_uint64), ("error_step", C.c_int32),
        ("kernel_launches", C.c_int32), ("device_seconds", C.c_double),
    ]


def sin_bench_problem(dim: int, kappa: float = 0.6, lam: float = 0.0,
                      horizon: float = 1.0) -> Problem:
    """make_problem(SinBenchmark{dim, kappa, lambda, horizon}) (benchmark.cpp:30-67)."""
    if lam <= 0.0:
        lam = 1.0 / math.sqrt(float(dim))  # SinBenchmark::lambda_value, benchmark.cpp:16-18
    p = Problem()
    p.dim = dim
    p.brownian_dim = dim
    p.horizon = horizon
    p.terminal_kind = TERMINAL_SIN_SUM
    p.driver_kind = DRIVER_SIN_BENCH
    p.drift_kind = DRIFT_ZERO
    p.diffusion_kind = DIFFUSION_IDENTITY
    p.terminal_params[0] = kappa
    p.terminal_params[1] = lam
    p.driver_params[0] = kappa
    p.driver_params[1] = lam
    p.growth_g = 2.0 + kappa
    p.growth_exp_g = 0.0
    p.growth_f = 1.0
    p.growth_exp_f = 0.0
    p.lipschitz_f = 2.0
    p.moment_ratio = 1.0
    p.state_bound = 1e15
    return p


def custom_problem(dim: int, terminal: int, driver: int, *, terminal_params=(), driver_params=(),
                   drift: int = DRIFT_ZERO, drift_params=(), diffusion: int = DIFFUSION_IDENTITY,
                   diffusion_params=(), horizon: float = 1.0, growth_g: float = 0.0,
                   growth_exp_g: float = 0.0, growth_f: float = 0.0, growth_exp_f: float = 0.0,
                   lipschitz_f: float = 0.0, moment_ratio: float = 1.0,
                   state_bound: float = 1e15, drift_vec=(), diffusion_vec=()) -> Problem:
    """A ProblemSpec built from device functor kinds (the test problems of
    proj/tests/test_solver.cpp:17-28 and acceptance_main.cpp:228-236)."""
    p = Problem()
    p.dim = dim
    p.brownian_dim = dim
    p.horizon = horizon
    p.terminal_kind = terminal
    p.driver_kind = driver
    p.drift_kind = drift
    p.diffusion_kind = diffusion
    for i, v in enumerate(terminal_params):
        p.terminal_params[i] = v
    for i, v in enumerate(driver_params):
        p.driver_params[i] = v
    for i, v in enumerate(drift_params):
        p.drift_params[i] = v
    for i, v in enumerate(diffusion_params):
        p.diffusion_params[i] = v
    for i, v in enumerate(drift_vec):  # AFFINE: [a_0..a_7, b_0..b_7], b_l(x) = a_l + b_l x_l
        p.drift_vec[i] = v
    for i, v in enumerate(diffusion_vec):  # DIAG: sigma_l
        p.diffusion_vec[i] = v
    p.growth_g, p.growth_exp_g, p.growth_f = growth_g, growth_exp_g, growth_f
    p.growth_exp_f, p.lipschitz_f = growth_exp_f, lipschitz_f
    p.moment_ratio, p.state_bound = moment_ratio, state_bound
    return p


class ConfigHolder:
    """Owns the arrays a Config points into (ctypes does not)."""

    def __init__(self, *, steps: int, paths: int, damping: float = 0.0, seed: int = 0,
                 workers: int = 0, memory_mode: int = MEMORY_STORE, gamma_kind: int = GAMMA_FULL,
                 degrees=(1,), mu: float = 2.0, center=None):
        self.degrees = (C.c_int32 * len(degrees))(*degrees)
        self.center = (C.c_double * len(center))(*center) if center is not None else None
        c = Config()
        c.steps = steps
        c.workers = workers
        c.paths = paths
        c.damping = damping
        c.seed = seed
        c.memory_mode = memory_mode
        c.gamma_kind = gamma_kind
        c.degrees = C.cast(self.degrees, C.POINTER(C.c_int32))
        c.n_degrees = len(degrees)
        c.mu = mu
        c.center = C.cast(self.center, C.POINTER(C.c_double)) if self.center is not None else None
        self.c = c

    def ref(self):
        return C.byref(self.c)


_LIB = None


def lib() -> C.CDLL:
    """The CUDA library. Raises if it is not built: there is no CPU fallback."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2407_21084_b200.build` "
                "(there is no CPU fallback)")
        _LIB = C.CDLL(str(LIB_PATH))
        _declare(_LIB)
    return _LIB


def _declare(L: C.CDLL) -> None:
    P, cp, sz = C.POINTER, C.c_char_p, C.c_size_t
    vp = C.c_void_p
    L.qrmc_problem_sin_bench.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_double, P(Problem)]
    L.qrmc_gpu_gamma_size.argtypes = [C.c_int32, C.c_int32, P(C.c_int32), C.c_int32]
    L.qrmc_gpu_gamma_size.restype = C.c_int64
    L.qrmc_gpu_gamma_indices.argtypes = [C.c_int32, C.c_int32, P(C.c_int32), C.c_int32,
                                         P(C.c_int32), sz, cp, sz]
    L.qrmc_gpu_session_create.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, P(vp), cp, sz]
    L.qrmc_gpu_session_destroy.argtypes = [vp]
    L.qrmc_gpu_session_destroy.restype = None
    L.qrmc_gpu_nccl_unique_id.argtypes = [vp, cp, sz]
    L.qrmc_gpu_backward_solve.argtypes = [vp, P(Problem), P(Config), P(C.c_double), sz,
                                          P(C.c_double), P(Stats), cp, sz]
    L.qrmc_gpu_plan_create.argtypes = [vp, P(Problem), P(Config), P(vp), cp, sz]
    L.qrmc_gpu_plan_run.argtypes = [vp, P(Stats), cp, sz]
    L.qrmc_gpu_plan_download.argtypes = [vp, P(C.c_double), sz, cp, sz]
    L.qrmc_gpu_plan_basis_size.argtypes = [vp]
    L.qrmc_gpu_plan_basis_size.restype = C.c_int64
    L.qrmc_gpu_plan_stream.argtypes = [vp]
    L.qrmc_gpu_plan_stream.restype = vp
    L.qrmc_gpu_plan_kernel_seconds.argtypes = [vp, P(C.c_double), P(C.c_double), cp, sz]
    L.qrmc_gpu_plan_io_bytes.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
    L.qrmc_gpu_mma_layout_check.argtypes = [C.c_int32, C.c_int32, P(C.c_int32), C.c_int32, C.c_uint64,
                                            P(C.c_int64), P(C.c_double), cp, sz]
    L.qrmc_gpu_plan_kernel_name.argtypes = [vp, C.c_int]
    L.qrmc_gpu_table_json.argtypes = [P(Config), C.c_int32, C.c_double, P(C.c_double), cp, sz, cp, sz]
    L.qrmc_gpu_table_json.restype = C.c_int64
    L.qrmc_gpu_plan_kernel_name.restype = C.c_char_p
    L.qrmc_gpu_lane_ownership.argtypes = [C.c_int64, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32),
                                          P(C.c_int64)]
    L.qrmc_gpu_replay_ranks_solve.argtypes = [P(Problem), P(Config), C.c_int32, P(C.c_double), sz, P(Stats), cp, sz]
    L.qrmc_gpu_owned_path.argtypes = [C.c_int64, C.c_int32, C.c_int32]
    L.qrmc_gpu_owned_path.restype = C.c_int64
    L.qrmc_gpu_plan_destroy.argtypes = [vp]
    L.qrmc_gpu_plan_destroy.restype = None
    L.qrmc_gpu_evaluate.argtypes = [P(Config), C.c_int32, P(C.c_double), P(C.c_double),
                                    C.c_int64, P(C.c_double), cp, sz]
    L.qrmc_gpu_mse_metrics.argtypes = [P(Config), C.c_int32, C.c_double, C.c_double, C.c_double,
                                       P(C.c_double), C.c_uint64, C.c_int32, P(C.c_double),
                                       P(C.c_double), cp, sz]
    L.qrmc_gpu_philox.argtypes = [P(C.c_uint32), P(C.c_uint32), C.c_int64, P(C.c_uint32), cp, sz]
    L.qrmc_gpu_stream_draws.argtypes = [C.c_uint64, P(C.c_uint64), C.c_int64, C.c_int32,
                                        C.c_int32, vp, cp, sz]
    L.qrmc_gpu_cloud_paths.argtypes = [P(Problem), P(Config), C.c_int32, C.c_int64, C.c_int64,
                                       P(C.c_double), cp, sz]


EXPORTED_SYMBOLS = (
    "qrmc_problem_sin_bench", "qrmc_gpu_gamma_size", "qrmc_gpu_gamma_indices",
    "qrmc_gpu_session_create", "qrmc_gpu_session_destroy", "qrmc_gpu_nccl_unique_id",
    "qrmc_gpu_backward_solve", "qrmc_gpu_plan_create", "qrmc_gpu_plan_run",
    "qrmc_gpu_plan_download", "qrmc_gpu_plan_basis_size", "qrmc_gpu_plan_stream",
    "qrmc_gpu_plan_kernel_seconds", "qrmc_gpu_plan_io_bytes", "qrmc_gpu_plan_kernel_name", "qrmc_gpu_mma_layout_check", "qrmc_gpu_table_json", "qrmc_gpu_lane_ownership",
    "qrmc_gpu_owned_path", "qrmc_gpu_replay_ranks_solve",
    "qrmc_gpu_plan_destroy", "qrmc_gpu_evaluate", "qrmc_gpu_mse_metrics", "qrmc_gpu_philox",
    "qrmc_gpu_stream_draws", "qrmc_gpu_cloud_paths",
)
