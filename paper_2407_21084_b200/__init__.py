"""B200-native backward solver for decoupled FBSDEs / semi-linear PDEs.

Drop-in for the reference's backward-induction loop ``qrmc::backward_solve``
(proj/src/solver.cpp:109-226): sm_100a CUDA kernels behind the C ABI in
include/qrmc_gpu.h, with a Python surface that mirrors the reference's
``qrmc`` bindings (proj/bindings/py_core.cpp). See DESIGN.md.
"""
from .api import (
    CapacityError,
    CoefficientTable,
    DeviceError,
    Measure,
    MetricReport,
    MultiIndexSet,
    NumericError,
    SimulationError,
    SinBenchmark,
    TruncationStats,
    backward_solve,
    confidence_interval,
    exact_solution,
    mse_metrics,
    solve,
)

__version__ = "0.1.0"
