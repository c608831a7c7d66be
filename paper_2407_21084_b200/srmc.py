"""Stratified regression Monte Carlo (SRMC) solver -- Python face of include/qrmc_srmc.h.

SURVEY.md 8(f) row f3: the north_star's hypercube/LP0/LP1/Z/Bergman features, which have
no code in the reference (parity unpinned; see include/qrmc_srmc.h for the scheme). The
problem/config objects keep the reference's plugin vocabulary: ``SinBenchmark`` functors
(proj/src/benchmark.cpp:30-67), ``RunConfig`` knobs steps/seed (proj/include/qrmc/
solver.hpp:24-35), the truncation bound (proj/src/solver.cpp:37-41). Everything runs in
``_lib/libqrmc_srmc.so`` (sm_100a); there is no CPU path -- a missing library raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("QRMC_SRMC_LIB", PKG_DIR / "_lib" / "libqrmc_srmc.so"))

SIN_BENCH, BERGMAN = 0, 1
LP0, LP1 = 0, 1
STATUS = {0: "OK", 1: "EINVAL", 2: "ENUMERIC", 3: "ESIM", 4: "ECAPACITY", 5: "ECUDA", 6: "ENCCL", 7: "ENOTIMPL"}


class SrmcProblem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_int32), ("horizon", C.c_double), ("params", C.c_double * 8)]


class SrmcConfig(C.Structure):
    _fields_ = [("steps", C.c_int32), ("cells_per_dim", C.c_int32), ("paths_per_cell", C.c_int64),
                ("basis", C.c_int32), ("want_z", C.c_int32), ("seed", C.c_uint64), ("lo", C.c_double),
                ("hi", C.c_double), ("truncation", C.c_double)]


class SrmcStats(C.Structure):
    _fields_ = [("path_steps", C.c_uint64), ("device_seconds", C.c_double), ("kernel_launches", C.c_int32),
                ("path_passes", C.c_int32)]


class SrmcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"SRMC CUDA library missing: {LIB_PATH} (run python -m paper_2407_21084_b200.build)")
        L = C.CDLL(str(LIB_PATH))
        P, Cf = C.POINTER(SrmcProblem), C.POINTER(SrmcConfig)
        dp = C.POINTER(C.c_double)
        L.qrmc_srmc_basis_size.argtypes = [P, Cf]
        L.qrmc_srmc_basis_size.restype = C.c_int32
        L.qrmc_srmc_cells.argtypes = [P, Cf]
        L.qrmc_srmc_cells.restype = C.c_int64
        L.qrmc_srmc_solve.argtypes = [P, Cf, dp, C.c_size_t, dp, C.c_size_t, C.POINTER(SrmcStats), C.c_char_p,
                                      C.c_size_t]
        L.qrmc_srmc_solve.restype = C.c_int32
        L.qrmc_srmc_evaluate.argtypes = [P, Cf, dp, dp, C.c_int64, dp, C.c_char_p, C.c_size_t]
        L.qrmc_srmc_evaluate.restype = C.c_int32
        vp = C.c_void_p
        L.qrmc_srmc_nccl_unique_id.argtypes = [vp, C.c_char_p, C.c_size_t]
        L.qrmc_srmc_nccl_unique_id.restype = C.c_int32
        L.qrmc_srmc_plan_create.argtypes = [P, Cf, C.c_int32, C.c_int32, C.c_int32, vp, C.c_int32, C.POINTER(vp),
                                            C.c_char_p, C.c_size_t]
        L.qrmc_srmc_plan_create.restype = C.c_int32
        L.qrmc_srmc_plan_run.argtypes = [vp, C.POINTER(SrmcStats), C.c_char_p, C.c_size_t]
        L.qrmc_srmc_plan_run.restype = C.c_int32
        L.qrmc_srmc_plan_download.argtypes = [vp, dp, C.c_size_t, dp, C.c_size_t, C.c_char_p, C.c_size_t]
        L.qrmc_srmc_plan_download.restype = C.c_int32
        L.qrmc_srmc_plan_stream.argtypes = [vp]
        L.qrmc_srmc_plan_stream.restype = vp
        L.qrmc_srmc_plan_destroy.argtypes = [vp]
        L.qrmc_srmc_plan_destroy.restype = None
        L.qrmc_srmc_cell_range.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.qrmc_srmc_cell_range.restype = C.c_int32
        _LIB = L
    return _LIB


def sin_bench_problem(d: int, kappa: float = 0.6, horizon: float = 1.0) -> SrmcProblem:
    """SinBenchmark(d, kappa, lambda = 1/sqrt(d), T) (proj/src/benchmark.cpp:16-18, 30-67)."""
    p = SrmcProblem(kind=SIN_BENCH, dim=d, horizon=horizon)
    p.params[0], p.params[1] = kappa, 1.0 / math.sqrt(d)
    return p


def sin_bench_exact(t: float, x: np.ndarray, kappa: float = 0.6, horizon: float = 1.0) -> np.ndarray:
    """u(t, x) = 1 + kappa + sin(lambda sum x) exp(lambda^2 d (t - T) / 2) (benchmark.cpp:20-28)."""
    x = np.atleast_2d(x)
    d = x.shape[1]
    lam = 1.0 / math.sqrt(d)
    return 1.0 + kappa + np.sin(lam * x.sum(axis=1)) * math.exp(lam * lam * d * (t - horizon) / 2.0)


def bergman_problem(d: int, mu: float, sigma: float, r_lend: float, r_borrow: float, strike: float,
                    horizon: float) -> SrmcProblem:
    """Bergman's different borrowing/lending rates (BASELINE config 3), d independent assets in
    log-price, payoff max(exp(mean x) - K, 0) (a geometric-basket call)."""
    p = SrmcProblem(kind=BERGMAN, dim=d, horizon=horizon)
    for j, v in enumerate((mu, sigma, r_lend, r_borrow, strike)):
        p.params[j] = v
    return p


def bergman_linear_exact(x0: np.ndarray, sigma: float, r: float, strike: float, horizon: float) -> float:
    """Black-Scholes price of the geometric-basket call when r_borrow == r_lend == r."""
    x0 = np.asarray(x0, dtype=float)
    d = x0.size
    m = x0.mean() + (r - 0.5 * sigma * sigma) * horizon
    v = sigma * sigma * horizon / d
    d2 = (m - math.log(strike)) / math.sqrt(v)
    d1 = d2 + math.sqrt(v)
    ncdf = lambda a: 0.5 * math.erfc(-a / math.sqrt(2.0))  # noqa: E731
    return math.exp(-r * horizon) * (math.exp(m + 0.5 * v) * ncdf(d1) - strike * ncdf(d2))


def config(steps: int, cells_per_dim: int, paths_per_cell: int, basis: int = LP1, lo: float = -4.0,
           hi: float = 4.0, truncation: float = 1e6, seed: int = 42, want_z: bool = False) -> SrmcConfig:
    return SrmcConfig(steps=steps, cells_per_dim=cells_per_dim, paths_per_cell=paths_per_cell, basis=basis,
                      want_z=int(want_z), seed=seed, lo=lo, hi=hi, truncation=truncation)


@dataclass
class SrmcTables:
    """y[i][k][P] and optionally z[i][k][l][P]; cells k lexicographic, coordinate d-1 fastest."""
    problem: SrmcProblem
    config: SrmcConfig
    y: np.ndarray
    z: np.ndarray | None
    stats: dict = field(default_factory=dict)

    def evaluate(self, step: int, x: np.ndarray) -> np.ndarray:
        """u(t_step, x) on the device (qrmc_srmc_evaluate)."""
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        out = np.empty(x.shape[0])
        tab = np.ascontiguousarray(self.y[step])
        err = C.create_string_buffer(256)
        dp = C.POINTER(C.c_double)
        rc = lib().qrmc_srmc_evaluate(C.byref(self.problem), C.byref(self.config), tab.ctypes.data_as(dp),
                                      x.ctypes.data_as(dp), x.shape[0], out.ctypes.data_as(dp), err, 256)
        if rc:
            raise SrmcError(rc, err.value.decode())
        return out


def solve(problem: SrmcProblem, cfg: SrmcConfig, with_z: bool = False) -> SrmcTables:
    """Full SRMC backward solve on the current CUDA device."""
    L = lib()
    P = L.qrmc_srmc_basis_size(C.byref(problem), C.byref(cfg))
    cells = L.qrmc_srmc_cells(C.byref(problem), C.byref(cfg))
    err = C.create_string_buffer(256)
    if P < 0 or cells < 0:
        # let the solve produce the precise validation message
        P, cells = max(P, 1), max(cells, 1)
    N, d = cfg.steps, problem.dim
    y = np.empty((N, cells, P))
    z = np.empty((N, cells, d, P)) if with_z else None
    st = SrmcStats()
    dp = C.POINTER(C.c_double)
    rc = L.qrmc_srmc_solve(C.byref(problem), C.byref(cfg), y.ctypes.data_as(dp), y.size,
                           z.ctypes.data_as(dp) if z is not None else None, z.size if z is not None else 0,
                           C.byref(st), err, 256)
    if rc:
        raise SrmcError(rc, err.value.decode())
    return SrmcTables(problem, cfg, y, z, {"path_steps": st.path_steps, "device_seconds": st.device_seconds,
                                          "kernel_launches": st.kernel_launches, "path_passes": st.path_passes})


class SrmcPlan:
    """qrmc_srmc_plan_* (include/qrmc_srmc.h): device-resident tables, the backward loop
    over this rank's hypercubes with an NCCL all-gather of every step's table when
    world > 1 (the library's own communicator; `nccl_id` comes from rank 0's
    ``nccl_unique_id()``, broadcast by the caller)."""

    def __init__(self, problem: SrmcProblem, cfg: SrmcConfig, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, keep_z: bool = False):
        L = lib()
        self.problem, self.config, self.world, self.rank = problem, cfg, world, rank
        self.handle = C.c_void_p()
        err = C.create_string_buffer(512)
        uid = (C.c_char * 128).from_buffer_copy(nccl_id) if nccl_id else None
        rc = L.qrmc_srmc_plan_create(C.byref(problem), C.byref(cfg), device, rank, world,
                                     C.cast(uid, C.c_void_p) if uid is not None else None, int(keep_z),
                                     C.byref(self.handle), err, 512)
        if rc:
            raise SrmcError(rc, err.value.decode())
        self.keep_z = keep_z

    def run(self) -> dict:
        st = SrmcStats()
        err = C.create_string_buffer(512)
        rc = lib().qrmc_srmc_plan_run(self.handle, C.byref(st), err, 512)
        if rc:
            raise SrmcError(rc, err.value.decode())
        return {"path_steps": st.path_steps, "device_seconds": st.device_seconds,
                "kernel_launches": st.kernel_launches, "path_passes": st.path_passes}

    def download(self, with_z: bool = False) -> SrmcTables:
        p, c = self.problem, self.config
        P = p.dim + 1 if c.basis == LP1 else 1
        cells = c.cells_per_dim ** p.dim
        y = np.empty((c.steps, cells, P))
        z = np.empty((c.steps, cells, p.dim, P)) if with_z else None
        dp = C.POINTER(C.c_double)
        err = C.create_string_buffer(512)
        rc = lib().qrmc_srmc_plan_download(self.handle, y.ctypes.data_as(dp), y.size,
                                           z.ctypes.data_as(dp) if z is not None else None,
                                           z.size if z is not None else 0, err, 512)
        if rc:
            raise SrmcError(rc, err.value.decode())
        return SrmcTables(p, c, y, z)

    def stream(self) -> int:
        return lib().qrmc_srmc_plan_stream(self.handle)

    def close(self) -> None:
        if self.handle:
            lib().qrmc_srmc_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    err = C.create_string_buffer(256)
    rc = lib().qrmc_srmc_nccl_unique_id(buf, err, 256)
    if rc:
        raise SrmcError(rc, err.value.decode())
    return bytes(buf)


def cell_range(cells: int, rank: int, world: int) -> tuple[int, int]:
    k0, k1 = C.c_int64(), C.c_int64()
    assert lib().qrmc_srmc_cell_range(cells, rank, world, C.byref(k0), C.byref(k1)) == 0
    return k0.value, k1.value


def _device_step_fn(problem: SrmcProblem, cfg: SrmcConfig):
    """step_fn for solve_sharded: qrmc_srmc_step_device on the current CUDA stream."""
    import torch
    L = lib()
    L.qrmc_srmc_step_device.argtypes = [C.POINTER(SrmcProblem), C.POINTER(SrmcConfig), C.c_int32, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_char_p,
                                        C.c_size_t]
    L.qrmc_srmc_step_device.restype = C.c_int32
    err = C.create_string_buffer(256)

    def step(i, nxt, y, z, k0, k1):
        rc = L.qrmc_srmc_step_device(C.byref(problem), C.byref(cfg), i, nxt.data_ptr() if nxt is not None else None,
                                     y.data_ptr(), z.data_ptr() if z is not None else None, k0, k1,
                                     torch.cuda.current_stream().cuda_stream, err, 256)
        if rc:
            raise SrmcError(rc, err.value.decode())
    return step


def solve_sharded(problem: SrmcProblem, cfg: SrmcConfig, with_z: bool = False, group=None, step_fn=None,
                  device=None) -> SrmcTables:
    """SRMC backward solve with the hypercubes partitioned over the ranks of ``group``
    (north_star item 5): rank r owns cells [r*c, min((r+1)*c, cells)), c = ceil(cells / G),
    runs each backward step on its cells only, and the step's y table is all-gathered
    (NCCL over NVLink on GPUs) before the next step, because paths land in arbitrary cells.
    Z is only read inside its own cell, so it is gathered once at the end (when asked for).
    Every cell's coefficients depend on nothing but (seed, step, cell) and the gathered
    table, so the result is bitwise identical for every G. ``step_fn(i, next, y, z, k0, k1)``
    defaults to the CUDA kernel; the CPU tests inject the oracle's per-range step."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if step_fn is None and (world == 1 or dist.get_backend(group) == "nccl"):
        # the library's plan: its own NCCL communicator all-gathers every step's table
        nid = None
        if world > 1:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            nid = obj[0]
        plan = SrmcPlan(problem, cfg, torch.cuda.current_device(), rank, world, nid, keep_z=with_z)
        try:
            st = plan.run()
            t = plan.download(with_z)
        finally:
            plan.close()
        k0, k1 = cell_range(cfg.cells_per_dim ** problem.dim, rank, world)
        t.stats = dict(st, cells=(k0, k1))
        return t
    d = problem.dim
    P = d + 1 if cfg.basis == LP1 else 1
    cells = cfg.cells_per_dim ** d
    per = -(-cells // world)
    rows = per * world
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if step_fn is None else torch.device("cpu")
    step_fn = step_fn or _device_step_fn(problem, cfg)
    N = cfg.steps
    needz = with_z or problem.kind == BERGMAN
    y = torch.zeros((N, rows, P), dtype=torch.float64, device=device)
    z = torch.zeros((N, rows, d, P), dtype=torch.float64, device=device) if needz else None
    k0, k1 = min(rank * per, cells), min((rank + 1) * per, cells)

    def gather(full: torch.Tensor) -> None:
        if world == 1:
            return
        mine = full[rank * per:(rank + 1) * per].clone()
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(full, mine, group=group)
        else:
            dist.all_gather(list(full.chunk(world)), mine, group=group)

    for i in range(N - 1, -1, -1):
        step_fn(i, y[i + 1] if i + 1 < N else None, y[i], z[i] if needz else None, k0, k1)
        gather(y[i])
    if with_z and world > 1:
        for i in range(N):
            gather(z[i])
    yh = y[:, :cells].cpu().numpy()
    zh = z[:, :cells].cpu().numpy() if with_z else None
    return SrmcTables(problem, cfg, yh, zh, {"path_steps": (k1 - k0) * cfg.paths_per_cell * N,
                                             "path_passes": 2 if problem.kind == BERGMAN else 1, "cells": (k0, k1)})
