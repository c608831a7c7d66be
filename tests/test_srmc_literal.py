"""SRMC replay parity at the LITERAL BASELINE.json config shapes (row f3; parity unpinned
against the reference, which has no SRMC code -- see include/qrmc_srmc.h).

A whole literal solve is far beyond what the CPU restatement finishes in seconds
(config 2: 40^4 cells x 1000 paths x 20 steps), so these tests replay single
backward steps on sampled cell ranges: the device kernel (qrmc_srmc_step_device)
and the restatement (oracle/srmc_oracle.c srmc_oracle_step) run the same step on
the same ranges of the full-size grid, reading the same step-(i+1) table (a
synthetic one: only its values matter, not how they were produced). Ranges sit at
the start, the middle and the end of the lexicographic cell order, so the cell
index arithmetic is exercised at every digit carry. Tolerance as in test_srmc.py:
|gpu - oracle| <= 1e-9 * max(1, max|oracle|).
"""
import ctypes as C
import math
import zlib

import numpy as np
import pytest

import oracles
from paper_2407_21084_b200 import srmc

pytestmark = pytest.mark.gpu
TOL = 1e-9
S0, K, T, SIG, MU = 100.0, 100.0, 0.5, 0.2, 0.05

LITERAL = [
    # BASELINE configs[1]: d=4 closed-form test, LP1, 40^4 hypercubes, N=20, M=1000
    ("config2-d4-lp1-40^4-M1000", lambda: srmc.sin_bench_problem(4),
     dict(steps=20, cells_per_dim=40, paths_per_cell=1000, basis=srmc.LP1), (19, 18, 0)),
    # BASELINE configs[2]: Bergman, d=4, LP1, N=20 (24^4 cells, M=500, Z pass + replay)
    ("config3-bergman-d4-lp1-24^4-M500",
     lambda: srmc.bergman_problem(4, MU, SIG, 0.01, 0.06, K, T),
     dict(steps=20, cells_per_dim=24, paths_per_cell=500, basis=srmc.LP1, lo=math.log(S0) - 0.6,
          hi=math.log(S0) + 0.6), (19, 7)),
    # BASELINE configs[3]: d=6, LP0, 16^6 ~ 1.7e7 hypercubes, N=10, M=100 (sub-warp hypercubes)
    ("config4-d6-lp0-16^6-M100", lambda: srmc.sin_bench_problem(6),
     dict(steps=10, cells_per_dim=16, paths_per_cell=100, basis=srmc.LP0), (9, 4)),
]
RANGE = 512


def ranges(cells):
    mid = cells // 2 - RANGE // 2
    return [(0, RANGE), (mid, mid + RANGE), (cells - RANGE, cells)]


def oracle_step_fn():
    o = oracles.srmc_port()
    Pp, Cp = C.POINTER(srmc.SrmcProblem), C.POINTER(srmc.SrmcConfig)
    dp = C.POINTER(C.c_double)
    o.L.srmc_oracle_step.argtypes = [Pp, Cp, C.c_int32, dp, dp, dp, C.c_int64, C.c_int64, C.c_int32]
    o.L.srmc_oracle_step.restype = C.c_int32
    return o.L.srmc_oracle_step


@pytest.mark.parametrize("name,mk,kw,steps", LITERAL, ids=[c[0] for c in LITERAL])
def test_literal_shape_steps_match_oracle_on_sampled_cells(name, mk, kw, steps):
    import torch
    p = mk()
    c = srmc.config(seed=2407, **kw)
    d = p.dim
    P = d + 1 if c.basis == srmc.LP1 else 1
    cells = c.cells_per_dim ** d
    needz = p.kind == srmc.BERGMAN
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    # a smooth-ish synthetic step-(i+1) table: level ~ the solution's scale plus small slopes
    base = 1.6 if p.kind == srmc.SIN_BENCH else 8.0
    nxt = np.empty((cells, P))
    nxt[:, 0] = base + 0.2 * rng.standard_normal(cells)
    if P > 1:
        nxt[:, 1:] = 0.05 * rng.standard_normal((cells, P - 1))
    nxt_dev = torch.from_numpy(nxt).cuda()
    y_dev = torch.zeros((cells, P), dtype=torch.float64, device="cuda")
    z_dev = torch.zeros((cells, d, P), dtype=torch.float64, device="cuda") if needz else None
    y_host = np.zeros((cells, P))
    z_host = np.zeros((cells, d, P)) if needz else None
    dev_step = srmc._device_step_fn(p, c)
    ora_step = oracle_step_fn()
    dp = C.POINTER(C.c_double)
    for i in steps:
        last = i == c.steps - 1
        for k0, k1 in ranges(cells):
            dev_step(i, None if last else nxt_dev, y_dev, z_dev, k0, k1)
            assert ora_step(C.byref(p), C.byref(c), i, None if last else nxt.ctypes.data_as(dp),
                            y_host.ctypes.data_as(dp), z_host.ctypes.data_as(dp) if needz else None, k0, k1, 0) == 0
        torch.cuda.synchronize()
        got_y = y_dev.cpu().numpy()
        for k0, k1 in ranges(cells):
            want = y_host[k0:k1]
            assert np.isfinite(want).all()
            scale = max(1.0, float(np.abs(want).max()))
            assert np.abs(got_y[k0:k1] - want).max() <= TOL * scale, (i, k0)
            if needz:
                got_z = z_dev.cpu().numpy()[k0:k1]
                zs = max(1.0, float(np.abs(z_host[k0:k1]).max()))
                assert np.abs(got_z - z_host[k0:k1]).max() <= TOL * zs, (i, k0)
        # cells outside the ranges are untouched (only the range is written)
        untouched = np.ones(cells, dtype=bool)
        for k0, k1 in ranges(cells):
            untouched[k0:k1] = False
        assert not got_y[untouched].any()
