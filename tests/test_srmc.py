"""SRMC solver (include/qrmc_srmc.h).

The reference has no SRMC code, so parity is UNPINNED against it. Two checks stand in:
* replay parity: GPU tables vs the C restatement oracle/srmc_oracle.c on the same Philox
  draws, |gpu - oracle| <= 1e-9 * max(1, max|oracle|) (FP64; only the reduction order
  differs), the cell index bit-exact;
* statistics: the solution against closed forms -- SinBenchmark's exact_solution
  (proj/src/benchmark.cpp:20-28) and Black-Scholes for the Bergman driver (linear case
  r_b = r_l; for a call the borrowing branch is always active, so the nonlinear price is
  Black-Scholes at r_b).
"""
import ctypes as C
import math

import numpy as np
import pytest

import oracles
from paper_2407_21084_b200 import srmc

TOL = 1e-9

# Bergman test market (Gobet-Lemor-Warin's call: S0 = K = 100, T = 0.5, mu = 5%, sigma = 20%)
S0, K, T, SIG, MU = 100.0, 100.0, 0.5, 0.2, 0.05


def _bergman(d, rl, rb):
    return srmc.bergman_problem(d, MU, SIG, rl, rb, K, T)


def _box(w=1.0):
    return math.log(S0) - w, math.log(S0) + w


# ------------------------------------------------------------------ CPU (no GPU)

def test_library_exports_and_host_validation():
    import re
    from pathlib import Path
    L = srmc.lib()
    text = (Path(__file__).resolve().parents[1] / "include" / "qrmc_srmc.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    declared = set(re.findall(r"\b(qrmc_srmc_\w+)\s*\(", text))
    assert declared == {"qrmc_srmc_basis_size", "qrmc_srmc_cells", "qrmc_srmc_solve", "qrmc_srmc_evaluate",
                        "qrmc_srmc_step_device", "qrmc_srmc_nccl_unique_id", "qrmc_srmc_plan_create",
                        "qrmc_srmc_plan_run", "qrmc_srmc_plan_download", "qrmc_srmc_plan_stream",
                        "qrmc_srmc_plan_destroy", "qrmc_srmc_cell_range"}
    for sym in declared:
        assert hasattr(L, sym), sym
    p = srmc.sin_bench_problem(3)
    c = srmc.config(4, 5, 64, basis=srmc.LP1)
    assert L.qrmc_srmc_basis_size(C.byref(p), C.byref(c)) == 4
    assert L.qrmc_srmc_cells(C.byref(p), C.byref(c)) == 125
    c0 = srmc.config(4, 5, 64, basis=srmc.LP0)
    assert L.qrmc_srmc_basis_size(C.byref(p), C.byref(c0)) == 1
    bad = srmc.config(4, 5, 3, basis=srmc.LP1)  # M < P
    assert L.qrmc_srmc_basis_size(C.byref(p), C.byref(bad)) == -1


def test_cell_range_partitions_the_hypercubes():
    for cells in (1, 7, 64, 4096, 16 ** 6):
        for world in (1, 2, 3, 4, 8):
            ranges = [srmc.cell_range(cells, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == cells
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(k1 - k0 for k0, k1 in ranges) - min(k1 - k0 for k0, k1 in ranges) <= -(-cells // world)


def test_plan_rejects_bad_input_before_touching_the_device():
    p = srmc.sin_bench_problem(2)
    with pytest.raises(srmc.SrmcError) as e:
        srmc.SrmcPlan(p, srmc.config(0, 4, 64))
    assert e.value.code == 1
    with pytest.raises(srmc.SrmcError) as e:
        srmc.SrmcPlan(p, srmc.config(3, 4, 64), rank=1, world=2)  # world > 1 without an NCCL id
    assert e.value.code == 1 and "NCCL" in str(e.value)
    with pytest.raises(srmc.SrmcError):
        srmc.SrmcPlan(p, srmc.config(1 << 22, 4, 64))  # stream-id layout (rng.hpp:73-80)


def test_srmc_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(srmc.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("mutate,code", [
    (lambda p, c: setattr(c, "paths_per_cell", 2), 1),
    (lambda p, c: setattr(c, "steps", 0), 1),
    (lambda p, c: setattr(c, "hi", c.lo), 1),
    (lambda p, c: setattr(c, "truncation", 0.0), 1),
    (lambda p, c: setattr(p, "kind", 9), 7),
    (lambda p, c: setattr(p, "dim", 7), 1),
    (lambda p, c: (setattr(c, "cells_per_dim", 2000), setattr(c, "paths_per_cell", 10**6)), 4),
])
def test_solve_rejects_bad_input_before_touching_the_device(mutate, code):
    p = srmc.sin_bench_problem(2)
    c = srmc.config(3, 4, 64)
    mutate(p, c)
    with pytest.raises(srmc.SrmcError) as e:
        srmc.solve(p, c)
    assert e.value.code == code


def test_oracle_sin_bench_converges_to_exact_solution():
    o = oracles.srmc_port()
    p = srmc.sin_bench_problem(1)
    c = srmc.config(10, 64, 8000, basis=srmc.LP1, lo=-4.0, hi=4.0)
    y, _ = o.solve(p, c)
    x = np.linspace(-2.0, 2.0, 41)[:, None]
    err = o.evaluate(p, c, y[0], x) - srmc.sin_bench_exact(0.0, x)
    assert np.abs(err).max() < 0.015, np.abs(err).max()


@pytest.mark.parametrize("rb", [0.01, 0.06])
def test_oracle_bergman_matches_black_scholes(rb):
    o = oracles.srmc_port()
    lo, hi = _box()
    p = _bergman(1, 0.01, rb)
    c = srmc.config(10, 127, 4000, basis=srmc.LP1, lo=lo, hi=hi)  # odd: x0 sits at a cell centre
    y, _ = o.solve(p, c)
    u = o.evaluate(p, c, y[0], np.array([[math.log(S0)]]))[0]
    bs = srmc.bergman_linear_exact([math.log(S0)], SIG, rb, K, T)
    assert abs(u - bs) < 0.02 * bs, (u, bs)


# ------------------------------------------------------------------ GPU

PARITY_CASES = [
    ("sin-d1-lp0", lambda: srmc.sin_bench_problem(1), dict(steps=5, cells_per_dim=16, paths_per_cell=45, basis=srmc.LP0)),
    ("sin-d2-lp1-z", lambda: srmc.sin_bench_problem(2), dict(steps=4, cells_per_dim=8, paths_per_cell=64, basis=srmc.LP1, want_z=True)),
    ("sin-d3-lp1", lambda: srmc.sin_bench_problem(3), dict(steps=3, cells_per_dim=5, paths_per_cell=37, basis=srmc.LP1)),
    # >= 32768 cells and M < 256: 4 lanes per hypercube (8 per warp), 33^3 leaves a tail group
    ("sin-d3-lp1-subwarp", lambda: srmc.sin_bench_problem(3), dict(steps=2, cells_per_dim=33, paths_per_cell=40, basis=srmc.LP1, want_z=True)),
    # M >= 256 without a Z pass also runs 4 lanes per hypercube (M < 2048)
    ("sin-d3-lp1-z-subwarp-m260", lambda: srmc.sin_bench_problem(3), dict(steps=2, cells_per_dim=33, paths_per_cell=260, basis=srmc.LP1, want_z=True)),
    ("bergman-d3-lp1-subwarp", lambda: _bergman(3, 0.01, 0.06), dict(steps=2, cells_per_dim=33, paths_per_cell=24, basis=srmc.LP1, lo=_box()[0], hi=_box()[1])),
    ("sin-d6-lp1-one-cell", lambda: srmc.sin_bench_problem(6), dict(steps=3, cells_per_dim=1, paths_per_cell=300, basis=srmc.LP1)),
    ("sin-d3-lp1-z-morton", lambda: srmc.sin_bench_problem(3), dict(steps=3, cells_per_dim=4, paths_per_cell=40, basis=srmc.LP1, want_z=True)),
    ("sin-d5-lp1-morton", lambda: srmc.sin_bench_problem(5), dict(steps=2, cells_per_dim=8, paths_per_cell=30, basis=srmc.LP1)),
    ("sin-d4-lp0-trunc", lambda: srmc.sin_bench_problem(4), dict(steps=3, cells_per_dim=4, paths_per_cell=33, basis=srmc.LP0, truncation=1.7)),
    ("bergman-d1-lp1", lambda: _bergman(1, 0.01, 0.06), dict(steps=5, cells_per_dim=32, paths_per_cell=100, basis=srmc.LP1, lo=_box()[0], hi=_box()[1])),
    ("bergman-d2-lp1", lambda: _bergman(2, 0.01, 0.06), dict(steps=4, cells_per_dim=8, paths_per_cell=96, basis=srmc.LP1, lo=_box()[0], hi=_box()[1])),
    ("bergman-d3-lp0", lambda: _bergman(3, 0.02, 0.05), dict(steps=3, cells_per_dim=4, paths_per_cell=50, basis=srmc.LP0, lo=_box()[0], hi=_box()[1])),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,mk,kw", PARITY_CASES, ids=[c[0] for c in PARITY_CASES])
def test_gpu_tables_match_oracle_on_replayed_draws(name, mk, kw):
    p = mk()
    c = srmc.config(seed=7, **kw)
    want_z = bool(kw.get("want_z")) or p.kind == srmc.BERGMAN
    got = srmc.solve(p, c, with_z=want_z)
    y, z = oracles.srmc_port().solve(p, c, with_z=want_z)
    scale = max(1.0, float(np.abs(y).max()))
    assert np.abs(got.y - y).max() <= TOL * scale
    if want_z:
        zs = max(1.0, float(np.abs(z).max()))
        assert np.abs(got.z - z).max() <= TOL * zs
    cells = c.cells_per_dim ** p.dim
    assert got.stats["path_steps"] == cells * c.paths_per_cell * c.steps
    assert got.stats["path_passes"] == (2 if p.kind == srmc.BERGMAN else 1)
    assert got.stats["kernel_launches"] == c.steps


@pytest.mark.gpu
@pytest.mark.parametrize("d,n", [(1, 7), (2, 16), (3, 9), (6, 4)])
def test_gpu_cell_index_bit_exact(d, n):
    """LP0 table holding its own cell number: evaluate() must return exactly the oracle's
    cell, for points inside, on cell faces and outside the box (projection)."""
    p = srmc.sin_bench_problem(d)
    c = srmc.config(1, n, 8, basis=srmc.LP0, lo=-1.3, hi=2.9)
    cells = n ** d
    tab = np.arange(cells, dtype=np.float64)[:, None]
    rng = np.random.default_rng(d * 100 + n)
    h = (c.hi - c.lo) / n
    x = np.concatenate([
        rng.uniform(c.lo - 1.0, c.hi + 1.0, (3000, d)),
        c.lo + h * rng.integers(0, n + 1, (1000, d)).astype(np.float64),  # exactly on faces
        np.full((1, d), c.lo), np.full((1, d), c.hi),
    ])
    tables = srmc.SrmcTables(p, c, tab[None], None)
    got = tables.evaluate(0, x)
    want = oracles.srmc_port().evaluate(p, c, tab, x)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_gpu_evaluate_matches_oracle_lp1():
    p = srmc.sin_bench_problem(3)
    c = srmc.config(3, 6, 64, basis=srmc.LP1)
    t = srmc.solve(p, c)
    x = np.random.default_rng(3).uniform(-5, 5, (500, 3))
    want = oracles.srmc_port().evaluate(p, c, t.y[0], x)
    assert np.abs(t.evaluate(0, x) - want).max() <= 1e-13


@pytest.mark.gpu
def test_gpu_sin_bench_d4_lp1_agrees_with_exact_solution():
    p = srmc.sin_bench_problem(4)
    c = srmc.config(10, 16, 1000, basis=srmc.LP1, lo=-4.0, hi=4.0)
    t = srmc.solve(p, c)
    x = np.random.default_rng(1).uniform(-1.5, 1.5, (400, 4))
    err = t.evaluate(0, x) - srmc.sin_bench_exact(0.0, x)
    assert np.abs(err).mean() < 0.01, np.abs(err).mean()
    assert np.abs(err).max() < 0.05, np.abs(err).max()


@pytest.mark.gpu
@pytest.mark.parametrize("rb", [0.01, 0.06])
def test_gpu_bergman_d4_agrees_with_black_scholes(rb):
    lo, hi = _box(0.6)
    p = _bergman(4, 0.01, rb)
    # odd cell count: x0 sits at a cell centre, where the LP1 fit is its (lowest-variance)
    # constant term; at a cell face the slope noise enters with weight 1
    c = srmc.config(10, 15, 4000, basis=srmc.LP1, lo=lo, hi=hi)
    t = srmc.solve(p, c, with_z=True)
    x0 = np.full((1, 4), math.log(S0))
    u = t.evaluate(0, x0)[0]
    bs = srmc.bergman_linear_exact(x0[0], SIG, rb, K, T)
    assert abs(u - bs) < 0.03 * bs, (u, bs)
    if rb > 0.01:  # the borrowing premium is visible
        assert u > srmc.bergman_linear_exact(x0[0], SIG, 0.01, K, T) + 0.5 * (bs - srmc.bergman_linear_exact(x0[0], SIG, 0.01, K, T))


@pytest.mark.gpu
@pytest.mark.parametrize("name,mk,kw", [PARITY_CASES[i] for i in (1, 3, 8)], ids=[PARITY_CASES[i][0] for i in (1, 3, 8)])
def test_gpu_per_range_steps_are_bitwise_equal_to_the_whole_solve(name, mk, kw):
    """qrmc_srmc_step_device over 3 uneven cell ranges per step (what 3 ranks of
    solve_sharded compute before their all-gather) == qrmc_srmc_solve, bit for bit; and
    solve_sharded at G=1 (no process group) == qrmc_srmc_solve."""
    import torch
    p = mk()
    c = srmc.config(seed=7, **kw)
    whole = srmc.solve(p, c, with_z=True)
    cells, d = c.cells_per_dim ** p.dim, p.dim
    P = whole.y.shape[2]
    y = torch.zeros((c.steps, cells, P), dtype=torch.float64, device="cuda")
    z = torch.zeros((c.steps, cells, d, P), dtype=torch.float64, device="cuda")
    step = srmc._device_step_fn(p, c)
    cuts = [0, cells // 5, cells // 5 + 1, cells]
    for i in range(c.steps - 1, -1, -1):
        for k0, k1 in zip(cuts[:-1], cuts[1:]):
            step(i, y[i + 1] if i + 1 < c.steps else None, y[i], z[i], k0, k1)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), whole.y)
    assert np.array_equal(z.cpu().numpy(), whole.z)
    g1 = srmc.solve_sharded(p, c, with_z=True)
    assert np.array_equal(g1.y, whole.y) and np.array_equal(g1.z, whole.z)


@pytest.mark.gpu
@pytest.mark.parametrize("name,mk,kw", [PARITY_CASES[i] for i in (1, 3, 8)], ids=[PARITY_CASES[i][0] for i in (1, 3, 8)])
def test_plan_runs_repeatably_and_equals_the_one_shot_solve(name, mk, kw):
    """qrmc_srmc_plan_*: the tables stay on the device across runs (allocated once) and
    every run reproduces qrmc_srmc_solve bit for bit."""
    p = mk()
    c = srmc.config(seed=7, **kw)
    whole = srmc.solve(p, c, with_z=True)
    plan = srmc.SrmcPlan(p, c, keep_z=True)
    try:
        for _ in range(2):
            st = plan.run()
            t = plan.download(with_z=True)
            assert np.array_equal(t.y, whole.y) and np.array_equal(t.z, whole.z)
            assert st["path_steps"] == c.cells_per_dim ** p.dim * c.paths_per_cell * c.steps
    finally:
        plan.close()


@pytest.mark.gpu
def test_plan_reports_non_finite_tables():
    p = srmc.sin_bench_problem(2)
    p.params[1] = float("nan")  # lambda = NaN: every coefficient non-finite
    with pytest.raises(srmc.SrmcError) as e:
        srmc.solve(p, srmc.config(3, 4, 64))
    assert e.value.code == 2


def test_ppnd16_split_branches_equal_the_whole():
    """The device evaluates PPND16's central rational per lane and batches the tails over
    the warp (srmc.cu srmc_quantiles) through qrmc_ppnd16_central / qrmc_ppnd16_tail;
    the two branches must reproduce qrmc_ppnd16 bit for bit (include/qrmc_normal_quantile.h)."""
    import ctypes as C
    o = oracles.srmc_port()
    f = o.L.srmc_oracle_ppnd16_both
    dp = C.POINTER(C.c_double)
    f.argtypes = [dp, C.c_int64, dp, dp]
    rng = np.random.default_rng(3)
    u = np.concatenate([rng.random(200_000), [0.075, 0.925, 0.5 - 0.425, 0.5 + 0.425, 1e-300, 1e-16, 1 - 2**-53,
                                              np.nextafter(0.075, 0), np.nextafter(0.925, 1), 2.0**-1074]])
    u = np.concatenate([u, np.exp(-rng.random(5000) * 700)])  # deep tails (r > 5 branch)
    whole, split = np.zeros_like(u), np.zeros_like(u)
    f(u.ctypes.data_as(dp), u.size, whole.ctypes.data_as(dp), split.ctypes.data_as(dp))
    np.testing.assert_array_equal(whole, split)


@pytest.mark.gpu
def test_gpu_bergman_path_cache_gives_the_same_tables(monkeypatch):
    """The Bergman second pass reads each path's (Y1, local coordinates) from a shared-memory
    cache written by the first pass (srmc.cu, M small enough); regenerating the path instead
    (QRMC_SRMC_PATH_CACHE=0) must give the same bits."""
    p = _bergman(4, 0.01, 0.06)
    lo, hi = _box()
    c = srmc.config(steps=3, cells_per_dim=6, paths_per_cell=300, basis=srmc.LP1, lo=lo, hi=hi, seed=5)
    a = srmc.solve(p, c, with_z=True)
    monkeypatch.setenv("QRMC_SRMC_PATH_CACHE", "0")
    b = srmc.solve(p, c, with_z=True)
    np.testing.assert_array_equal(a.y, b.y)
    np.testing.assert_array_equal(a.z, b.z)
