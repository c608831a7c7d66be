"""Test-side loaders for the two CPU oracles (TEST INFRASTRUCTURE ONLY).

* ``port()`` -- oracle/lib/libqrmc_oracle.so, the plain-C restatement
  (oracle/qrmc_oracle.c), symbols ``qrmc_orc_*``.
* ``ref()``  -- oracle/_ref/libqrmc_ref.so, the unmodified reference sources
  plus the Boost shim (oracle/Makefile), symbols ``qrmc_ref_*``. Present only
  where it was built (this container; it also travels to GPU boxes inside the
  repo snapshot).

Both expose the same calls with the C structs of include/qrmc_gpu.h, so the
parity tests can hold the GPU library, the port and the reference side by side.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2407_21084_b200 import _abi

ROOT = Path(__file__).resolve().parents[1]
PORT_PATH = ROOT / "oracle" / "lib" / "libqrmc_oracle.so"
REF_PATH = ROOT / "oracle" / "_ref" / "libqrmc_ref.so"

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_abi.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Oracle:
    def __init__(self, path: Path, prefix: str):
        self.path = path
        self.prefix = prefix
        self.L = C.CDLL(str(path))
        P, sz, cp = C.POINTER, C.c_size_t, C.c_char_p
        f = self._f
        f("philox").argtypes = [P(C.c_uint32), P(C.c_uint32), C.c_int64, P(C.c_uint32)]
        f("stream_draws").argtypes = [C.c_uint64, P(C.c_uint64), C.c_int64, C.c_int32, C.c_int32,
                                      C.c_void_p]
        f("normal_quantile").argtypes = [C.c_double]
        f("normal_quantile").restype = C.c_double
        f("measure").argtypes = [C.c_double, C.c_int32, _dp, C.c_int32, C.c_int32, _dp, C.c_int64,
                                 _dp, cp, sz]
        f("gamma_size").argtypes = [C.c_int32, C.c_int32, P(C.c_int32), C.c_int32]
        f("gamma_size").restype = C.c_int64
        f("gamma_indices").argtypes = [C.c_int32, C.c_int32, P(C.c_int32), C.c_int32,
                                       P(C.c_int32), sz, P(C.c_int32), cp, sz]
        f("backward_solve").argtypes = [P(_abi.Problem), P(_abi.Config), _dp, sz, _dp,
                                        P(_abi.Stats), cp, sz]
        f("cloud_paths").argtypes = [P(_abi.Problem), P(_abi.Config), C.c_int32, C.c_int64,
                                     C.c_int64, _dp, cp, sz]
        f("response").argtypes = [P(_abi.Problem), P(_abi.Config), _dp, P(C.c_uint8), C.c_int32,
                                  _dp, C.c_int64, _dp, P(C.c_uint64), P(C.c_uint64), cp, sz]
        f("eval_series").argtypes = [P(_abi.Config), C.c_int32, _dp, _dp, C.c_int64, _dp, cp, sz]
        f("evaluate").argtypes = [P(_abi.Config), C.c_int32, _dp, _dp, C.c_int64, _dp, cp, sz]
        f("mse_metrics").argtypes = [P(_abi.Config), C.c_int32, C.c_double, C.c_double,
                                     C.c_double, _dp, C.c_uint64, C.c_int32, _dp, _dp, cp, sz]
        if prefix == "qrmc_orc_":
            f("backward_solve_lanes").argtypes = [P(_abi.Problem), P(_abi.Config), _dp, sz,
                                                  C.c_int32, C.c_int32, _dp, P(_abi.Stats), cp, sz]

    def _f(self, name):
        return getattr(self.L, self.prefix + name)

    @staticmethod
    def _check(rc, err):
        if rc != 0:
            raise OracleError(rc, err.value.decode(errors="replace"))

    # ------------------------------------------------------------------ rng
    def philox(self, ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
        ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
        key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
        out = np.zeros_like(ctr)
        self._f("philox")(_ptr(ctr, C.c_uint32), _ptr(key, C.c_uint32), len(ctr),
                          _ptr(out, C.c_uint32))
        return out

    def stream_draws(self, seed: int, sids, n_draws: int, kind: int) -> np.ndarray:
        sids = np.ascontiguousarray(sids, dtype=np.uint64)
        out = np.zeros((len(sids), n_draws), dtype=np.uint64 if kind == 0 else np.float64)
        self._f("stream_draws")(seed, _ptr(sids, C.c_uint64), len(sids), n_draws, kind,
                                out.ctypes.data_as(C.c_void_p))
        return out

    def normal_quantile(self, p: float) -> float:
        return self._f("normal_quantile")(p)

    def measure(self, mu, dim, op, x, coord=0, center=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros_like(x)
        cen = None if center is None else np.ascontiguousarray(center, dtype=np.float64)
        err = C.create_string_buffer(512)
        rc = self._f("measure")(mu, dim, None if cen is None else _ptr(cen), op, coord, _ptr(x),
                                x.size, _ptr(out), err, 512)
        self._check(rc, err)
        return out

    # ---------------------------------------------------------------- gamma
    def gamma(self, kind: int, dim: int, degrees) -> tuple[np.ndarray, np.ndarray]:
        deg = (C.c_int32 * len(degrees))(*degrees)
        n = self._f("gamma_size")(kind, dim, deg, len(degrees))
        if n < 0:
            raise OracleError(-n, "gamma_size")
        rows = np.zeros((n, dim), dtype=np.int32)
        kmax = np.zeros(dim, dtype=np.int32)
        err = C.create_string_buffer(512)
        rc = self._f("gamma_indices")(kind, dim, deg, len(degrees), _ptr(rows, C.c_int32),
                                      rows.size, _ptr(kmax, C.c_int32), err, 512)
        self._check(rc, err)
        return rows, kmax

    # --------------------------------------------------------------- solver
    def backward_solve(self, problem: _abi.Problem, cfg: _abi.ConfigHolder, basis_size: int):
        coeffs = np.zeros((cfg.c.steps, basis_size))
        wall = np.zeros(cfg.c.steps)
        stats = _abi.Stats()
        err = C.create_string_buffer(1024)
        rc = self._f("backward_solve")(C.byref(problem), cfg.ref(), _ptr(coeffs), coeffs.size,
                                       _ptr(wall), C.byref(stats), err, 1024)
        self._check(rc, err)
        return coeffs, stats

    def backward_solve_status(self, problem, cfg, basis_size):
        coeffs = np.zeros((cfg.c.steps, basis_size))
        stats = _abi.Stats()
        err = C.create_string_buffer(1024)
        rc = self._f("backward_solve")(C.byref(problem), cfg.ref(), _ptr(coeffs), coeffs.size,
                                       None, C.byref(stats), err, 1024)
        return rc, stats, err.value.decode()

    def backward_solve_lanes(self, problem, cfg, basis_size, lane_lo, lane_hi):
        coeffs = np.zeros((cfg.c.steps, basis_size))
        part = np.zeros((lane_hi - lane_lo, basis_size))
        stats = _abi.Stats()
        err = C.create_string_buffer(1024)
        rc = self._f("backward_solve_lanes")(C.byref(problem), cfg.ref(), _ptr(coeffs),
                                             coeffs.size, lane_lo, lane_hi, _ptr(part),
                                             C.byref(stats), err, 1024)
        self._check(rc, err)
        return coeffs, part

    def cloud_paths(self, problem, cfg, step: int, first: int, n: int) -> np.ndarray:
        d = problem.dim
        out = np.zeros((n, cfg.c.steps - step + 1, d))
        err = C.create_string_buffer(512)
        rc = self._f("cloud_paths")(C.byref(problem), cfg.ref(), step, first, n, _ptr(out), err,
                                    512)
        self._check(rc, err)
        return out

    def response(self, problem, cfg, coeffs, have_step, start, paths):
        paths = np.ascontiguousarray(paths, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        have = np.ascontiguousarray(have_step, dtype=np.uint8)
        out = np.zeros(paths.shape[0])
        apps, clip = C.c_uint64(), C.c_uint64()
        err = C.create_string_buffer(512)
        rc = self._f("response")(C.byref(problem), cfg.ref(), _ptr(coeffs),
                                 _ptr(have, C.c_uint8), start, _ptr(paths), paths.shape[0],
                                 _ptr(out), C.byref(apps), C.byref(clip), err, 512)
        self._check(rc, err)
        return out, apps.value, clip.value

    def eval_series(self, cfg, dim, coeffs_step, x):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, dim)
        c = np.ascontiguousarray(coeffs_step, dtype=np.float64)
        out = np.zeros(x.shape[0])
        err = C.create_string_buffer(512)
        rc = self._f("eval_series")(cfg.ref(), dim, _ptr(c), _ptr(x), x.shape[0], _ptr(out),
                                    err, 512)
        self._check(rc, err)
        return out

    def evaluate(self, cfg, dim, coeffs_step, x):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, dim)
        c = np.ascontiguousarray(coeffs_step, dtype=np.float64)
        out = np.zeros(x.shape[0])
        err = C.create_string_buffer(512)
        rc = self._f("evaluate")(cfg.ref(), dim, _ptr(c), _ptr(x), x.shape[0], _ptr(out), err,
                                 512)
        self._check(rc, err)
        return out

    def mse_metrics(self, cfg, dim, kappa, lam, horizon, coeffs, eval_seed, eval_points=1000):
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros(6)
        step_sq = np.zeros(cfg.c.steps)
        err = C.create_string_buffer(512)
        rc = self._f("mse_metrics")(cfg.ref(), dim, kappa, lam, horizon, _ptr(c), eval_seed,
                                    eval_points, _ptr(out), _ptr(step_sq), err, 512)
        self._check(rc, err)
        return out, step_sq


_cache: dict[str, Oracle] = {}


def port() -> Oracle:
    if "port" not in _cache:
        if not PORT_PATH.exists():
            raise RuntimeError(f"{PORT_PATH} missing: run `make -C oracle port`")
        _cache["port"] = Oracle(PORT_PATH, "qrmc_orc_")
    return _cache["port"]


def have_ref() -> bool:
    return REF_PATH.exists()


def ref() -> Oracle:
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_PATH, "qrmc_ref_")
    return _cache["ref"]


SRMC_PATH = ROOT / "oracle" / "lib" / "libsrmc_oracle.so"


class SrmcOracle:
    """oracle/srmc_oracle.c: CPU restatement of the SRMC scheme (include/qrmc_srmc.h).
    Parity unpinned against the reference (no SRMC code there); checker only."""

    def __init__(self, path: Path):
        from paper_2407_21084_b200 import srmc
        self.srmc = srmc
        self.L = C.CDLL(str(path))
        Pp, Cp = C.POINTER(srmc.SrmcProblem), C.POINTER(srmc.SrmcConfig)
        self.L.srmc_oracle_solve.argtypes = [Pp, Cp, _dp, _dp, C.c_int32]
        self.L.srmc_oracle_solve.restype = C.c_int32
        self.L.srmc_oracle_eval.argtypes = [Pp, Cp, _dp, _dp]
        self.L.srmc_oracle_eval.restype = C.c_double

    def solve(self, prob, cfg, with_z: bool = False, threads: int = 0):
        d = prob.dim
        P = d + 1 if cfg.basis == self.srmc.LP1 else 1
        cells = cfg.cells_per_dim ** d
        y = np.zeros((cfg.steps, cells, P))
        z = np.zeros((cfg.steps, cells, d, P)) if with_z else None
        rc = self.L.srmc_oracle_solve(C.byref(prob), C.byref(cfg), _ptr(y), _ptr(z) if z is not None else None,
                                      threads)
        assert rc == 0
        return y, z

    def evaluate(self, prob, cfg, y_step: np.ndarray, x: np.ndarray) -> np.ndarray:
        y_step = np.ascontiguousarray(y_step, dtype=np.float64)
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float64)
        return np.array([self.L.srmc_oracle_eval(C.byref(prob), C.byref(cfg), _ptr(y_step), _ptr(row))
                         for row in x])


def srmc_port() -> SrmcOracle:
    if "srmc" not in _cache:
        if not SRMC_PATH.exists():
            raise RuntimeError(f"{SRMC_PATH} missing: run `make -C oracle port`")
        _cache["srmc"] = SrmcOracle(SRMC_PATH)
    return _cache["srmc"]


def srmc_oracle_step_fn(prob, cfg, threads: int = 1):
    """step_fn for srmc.solve_sharded on CPU tensors: the oracle's per-range step."""
    o = srmc_port()
    Pp, Cp = C.POINTER(o.srmc.SrmcProblem), C.POINTER(o.srmc.SrmcConfig)
    o.L.srmc_oracle_step.argtypes = [Pp, Cp, C.c_int32, _dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int32]
    o.L.srmc_oracle_step.restype = C.c_int32

    def step(i, nxt, y, z, k0, k1):
        p = lambda t: C.cast(t.data_ptr(), _dp) if t is not None else None  # noqa: E731
        assert o.L.srmc_oracle_step(C.byref(prob), C.byref(cfg), i, p(nxt), p(y), p(z), k0, k1, threads) == 0
    return step
