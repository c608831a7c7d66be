"""Command-line front end with the reference CLI's subcommands and flags
(proj/tools/qrmc_main.cpp), running the solve on the B200 library.

    python -m paper_2407_21084_b200 solve --dim 4 --kind hyperbolic --deg 16 --steps 20 \\
        --paths 1000000 --q 5.1 --seed 42 --out table.json
    python -m paper_2407_21084_b200 bench --dim 4 ... --runs 5 --out report.json
    python -m paper_2407_21084_b200 mindex-card --dim 6 --kind hyperbolic --deg 64

Exit codes follow qrmc_main.cpp:36-39,351-370: 0 ok, 1 usage / capacity, 2 numeric or
simulation error, 3 I/O error. Artifacts: `--out` of `solve` writes the reference's
byte-identical `qrmc.coefficients.v1` document (table_io.cpp:45-81) plus a
`.meta.json` run record (table_io.cpp:138-159); `bench --out` writes the
`qrmc.metrics.v1` report (benchmark.cpp:188-221) as JSON or CSV.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time

import numpy as np

from . import api

EXIT_OK, EXIT_USAGE, EXIT_NUMERIC, EXIT_IO = 0, 1, 2, 3


def _positive(kind):
    def conv(s):
        v = kind(s)
        if not v > 0:
            raise argparse.ArgumentTypeError(f"{s} is not positive")
        return v
    return conv


def _nonneg(kind):
    def conv(s):
        v = kind(s)
        if v < 0:
            raise argparse.ArgumentTypeError(f"{s} is negative")
        return v
    return conv


def _add_solve_flags(p: argparse.ArgumentParser) -> None:
    """add_solve_flags (qrmc_main.cpp:56-103)."""
    p.add_argument("--dim", type=_positive(int), required=True, help="State dimension d")
    p.add_argument("--mu", type=_positive(float), default=2.0, help="Student shape parameter")
    p.add_argument("--center", type=float, nargs="+", default=None, help="Sampling measure center (d values)")
    p.add_argument("--q", type=_nonneg(float), default=0.0, dest="damping", help="Damping exponent q >= 0")
    p.add_argument("--steps", type=_positive(int), required=True, help="Time steps N")
    p.add_argument("--kind", choices=["full", "total", "hyperbolic"], default="full", help="Index set kind")
    p.add_argument("--deg", type=_nonneg(int), default=0, dest="degree", help="Degree parameter")
    p.add_argument("--degrees", type=int, nargs="+", default=None, help="Per-coordinate degrees (full only)")
    p.add_argument("--paths", type=_positive(int), required=True, help="Monte-Carlo paths per step M")
    p.add_argument("--seed", type=int, default=0, help="Base seed")
    p.add_argument("--threads", "--workers", type=_nonneg(int), default=0, dest="workers",
                   help="Worker threads (accepted for compatibility; the device sets its own)")
    p.add_argument("--memory-mode", choices=["store", "recompute"], default="store")
    p.add_argument("--kappa", type=float, default=0.6, help="Benchmark offset kappa")
    p.add_argument("--lambda", type=_nonneg(float), default=0.0, dest="lambda_",
                   help="Benchmark frequency lambda (0 = 1/sqrt(d))")
    p.add_argument("--horizon", type=_positive(float), default=1.0, help="Terminal time T")


class _UsageError(Exception):
    pass


def _gamma(o) -> api.MultiIndexSet:
    """build_gamma (qrmc_main.cpp:105-117)."""
    if o.degrees:
        if o.kind != "full":
            raise _UsageError("--degrees: per-coordinate degrees are only valid with --kind full")
        if len(o.degrees) != o.dim:
            raise _UsageError("--degrees: need exactly d values")
        return api.MultiIndexSet.full(o.degrees)
    if o.kind == "full":
        return api.MultiIndexSet.full([o.degree] * o.dim)
    return api.MultiIndexSet(o.kind, o.dim, (o.degree,))


def _bench(o) -> api.SinBenchmark:
    lam = o.lambda_ if o.lambda_ > 0 else 1.0 / math.sqrt(o.dim)
    return api.SinBenchmark(dim=o.dim, kappa=o.kappa, lambda_=lam, horizon=o.horizon)


def _measure(o) -> api.Measure:
    return api.Measure(o.mu, o.dim, tuple(o.center) if o.center else ())


def _christoffel(gamma: api.MultiIndexSet) -> float:
    """christoffel_number (cosine_basis.cpp:30-39): sum over Gamma of 2^nnz(k)."""
    rows = gamma.indices()
    return float(np.sum(np.ldexp(1.0, np.count_nonzero(rows, axis=1))))


def _summary(gamma, paths) -> None:
    c = _christoffel(gamma)
    print(f"basis size {len(gamma)}, christoffel {c:.6g}, statistical indicator "
          f"christoffel/M = {c / paths:.6g}")


def run_solve(o) -> int:
    """run_solve (qrmc_main.cpp:146-172)."""
    gamma = _gamma(o)
    _summary(gamma, o.paths)
    if o.dry_run:
        m, k = o.paths, len(gamma)
        b = m * 8 + (m * o.dim * 8 if o.memory_mode == "store" else 0) + 256 * k * 8 + o.steps * k * 8
        print(f"dry run: memory estimate {b / (1024.0 * 1024.0):.1f} MiB, no simulation performed")
        return EXIT_OK
    table = api.solve(_bench(o), gamma, _measure(o), o.steps, o.paths, o.damping, o.seed, o.workers,
                      o.memory_mode)
    if o.out:
        table.save_json(o.out)
        wall = [float(s) for s in (table.step_wall_seconds if table.step_wall_seconds is not None else [])]
        meta = {"schema": "qrmc.run_meta.v1", "memory_mode": o.memory_mode, "workers": o.workers,
                "wall_seconds_per_step": wall, "total_wall_seconds": float(sum(wall)),
                "truncation": {"applications": table.truncation.applications,
                               "clipped": table.truncation.clipped},
                "unix_time": int(time.time())}
        with open(o.out + ".meta.json", "w") as f:
            f.write(json.dumps(meta, indent=2) + "\n")
        print(f"wrote {o.out} (+ .meta.json)")
    print(f"value at origin, t=0: {table.evaluate(0, np.zeros(o.dim)):.6f}")
    return EXIT_OK


def _fmt(v: float) -> str:
    """format_double (benchmark.cpp:178-184): 10 significant digits, %g style."""
    if not math.isfinite(v):
        return "inf" if v > 0 else "-inf"
    return f"{v:.10g}"


def _report_json(r: dict) -> str:
    def fin(v):
        return v if math.isfinite(v) else ("inf" if v > 0 else "-inf")
    doc = {"schema": "qrmc.metrics.v1", "mse_max": fin(r["mse_max"]), "mse_av": fin(r["mse_av"]),
           "mse_max_undamped": fin(r["mse_max_undamped"]), "mse_av_undamped": fin(r["mse_av_undamped"]),
           "eval_points_per_step": r["eval_points_per_step"], "step_squared_error": r["step_squared_error"],
           "dim": r["dim"], "delta": r["delta"], "damping": r["damping"], "kind": r["kind"],
           "degree": r["degree"], "basis_size": r["basis_size"], "paths": r["paths"], "seed": r["seed"],
           "stat_error_indicator": r["stat_error_indicator"], "wall_seconds": r["wall_seconds"]}
    return json.dumps(doc, indent=2)


def _report(table: api.CoefficientTable, bench: api.SinBenchmark, eval_seed: int, eval_points: int,
            wall: float) -> dict:
    m = api.mse_metrics(table, bench, eval_seed, eval_points)
    g = table.gamma
    return {"mse_max": float(m.mse_max), "mse_av": float(m.mse_av), "mse_max_undamped": float(m.mse_max_undamped),
            "mse_av_undamped": float(m.mse_av_undamped), "eval_points_per_step": eval_points,
            "step_squared_error": [float(v) for v in m.step_squared_error], "dim": g.dim, "delta": table.dt(),
            "damping": table.damping, "kind": g.kind, "degree": int(g.degrees[0]) if g.degrees else 0,
            "basis_size": len(g), "paths": table.paths, "seed": table.seed,
            "stat_error_indicator": _christoffel(g) / table.paths, "wall_seconds": wall}


def run_bench(o) -> int:
    """run_bench (qrmc_main.cpp:174-234)."""
    bench = _bench(o)
    reports, origin = [], []
    if o.table:
        table = api.CoefficientTable.load_json(o.table)
        reports.append(_report(table, bench, o.eval_seed, o.eval_points, 0.0))
        origin.append(table.evaluate(0, np.zeros(o.dim)))
    else:
        gamma = _gamma(o)
        _summary(gamma, o.paths)
        for r in range(o.runs):
            seed = o.seed + r
            t0 = time.perf_counter()
            table = api.solve(bench, gamma, _measure(o), o.steps, o.paths, o.damping, seed, o.workers,
                              o.memory_mode)
            wall = time.perf_counter() - t0
            rep = _report(table, bench, o.eval_seed, o.eval_points, wall)
            origin.append(table.evaluate(0, np.zeros(o.dim)))
            print(f"run {r} (seed {seed}): mse_max {rep['mse_max']:.4f}, mse_av {rep['mse_av']:.4f}, "
                  f"y(0) {origin[-1]:.5f}, {wall:.2f}s")
            reports.append(rep)
    if len(origin) >= 2:
        lo, hi = api.confidence_interval(origin, 0.99)
        print(f"99% CI of value at origin over {len(origin)} runs: [{lo:.5f}, {hi:.5f}]")
    if o.out:
        with open(o.out, "w") as f:
            if o.format == "csv":
                f.write("d,delta,q,kind,degree,basis_size,paths,seed,mse_max,mse_av,wall_seconds\n")
                for r in reports:
                    f.write(",".join([str(r["dim"]), _fmt(r["delta"]), _fmt(r["damping"]), r["kind"],
                                      str(r["degree"]), str(r["basis_size"]), str(r["paths"]), str(r["seed"]),
                                      _fmt(r["mse_max"]), _fmt(r["mse_av"]), _fmt(r["wall_seconds"])]) + "\n")
            else:
                f.write("[\n" + ",\n".join(_report_json(r) for r in reports) + "\n]\n")
        print(f"wrote {o.out}")
    return EXIT_OK


def run_mindex_card(o) -> int:
    print(len(api.MultiIndexSet.full([o.deg] * o.dim) if o.kind == "full" else api.MultiIndexSet(o.kind, o.dim, (o.deg,))))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="qrmc-gpu", description="Quasi-regression Monte Carlo solver for decoupled "
                                 "Markovian BSDEs / semi-linear parabolic PDEs (B200 backend)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    ps = sub.add_parser("solve", help="Backward-solve the benchmark problem, write coefficients")
    _add_solve_flags(ps)
    ps.add_argument("--dry-run", action="store_true")
    ps.add_argument("--out", default="", help="Coefficient artifact path (JSON)")
    pb = sub.add_parser("bench", help="Solve and score against the closed-form solution")
    _add_solve_flags(pb)
    pb.add_argument("--runs", type=_positive(int), default=1)
    pb.add_argument("--eval-seed", type=int, default=0x9E3779B97F4A7C15)
    pb.add_argument("--eval-points", type=_positive(int), default=1000)
    pb.add_argument("--table", default="", help="Score an existing coefficient artifact instead of solving")
    pb.add_argument("--out", default="")
    pb.add_argument("--format", choices=["json", "csv"], default="json")
    pc = sub.add_parser("mindex-card", help="Print a multi-index set cardinality")
    pc.add_argument("--dim", type=_positive(int), required=True)
    pc.add_argument("--kind", choices=["full", "total", "hyperbolic"], default="total")
    pc.add_argument("--deg", type=_nonneg(int), required=True)
    try:
        o = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        if o.cmd == "solve":
            return run_solve(o)
        if o.cmd == "bench":
            return run_bench(o)
        return run_mindex_card(o)
    except _UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except OSError as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except api.NumericError as e:
        print(f"numeric error: {e}", file=sys.stderr)
        return EXIT_NUMERIC
    except api.SimulationError as e:
        print(f"simulation error: {e}", file=sys.stderr)
        return EXIT_NUMERIC
    except api.CapacityError as e:
        print(f"capacity error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except ValueError as e:
        msg = str(e)
        if msg.startswith("coefficient artifact"):
            print(f"I/O error: {msg}", file=sys.stderr)
            return EXIT_IO
        print(f"error: {msg}", file=sys.stderr)
        return EXIT_USAGE
