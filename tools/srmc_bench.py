"""SRMC throughput on one B200 (BASELINE.json configs 2-4 in their
literal hypercube form -- the reference cannot run them, so there is no reference arm).

    python tools/srmc_bench.py [--quick] [--ncu]

One JSON line per workload: path-steps/s from the CUDA-event time of the solve's kernels
(`device`), and end to end through srmc.solve() including the device->host copy of every
table (`e2e`). Inputs are generated on the device by the counter-based stream, so there is
no host->device traffic. A path-step = one (cell, path) Euler step with its gather and
normal-equation update; a Z pass (Bergman) counts again.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_21084_b200 import srmc  # noqa: E402

WORKLOADS = {
    # BASELINE config 2: d=4, LP1, 40^4 hypercubes, N=20, M=1000 paths/cell
    "c2-sin-d4-lp1-40^4-N20-M1000": (lambda: srmc.sin_bench_problem(4),
                                     dict(steps=20, cells_per_dim=40, paths_per_cell=1000, basis=srmc.LP1)),
    # BASELINE config 3: Bergman, d=4, LP1, N=20 (cells/paths chosen here: 24^4, M=500)
    "c3-bergman-d4-lp1-24^4-N20-M500": (
        lambda: srmc.bergman_problem(4, 0.05, 0.2, 0.01, 0.06, 100.0, 0.5),
        dict(steps=20, cells_per_dim=24, paths_per_cell=500, basis=srmc.LP1, lo=math.log(100) - 0.6,
             hi=math.log(100) + 0.6)),
    # BASELINE config 4 on one GPU: d=6, LP0, 16^6 = 1.7e7 hypercubes, N=10 (M=100 paths/cell)
    "c4-sin-d6-lp0-16^6-N10-M100": (lambda: srmc.sin_bench_problem(6),
                                    dict(steps=10, cells_per_dim=16, paths_per_cell=100, basis=srmc.LP0)),
}
QUICK = {"c2q-sin-d4-lp1-40^4-N2-M1000": (lambda: srmc.sin_bench_problem(4),
                                         dict(steps=2, cells_per_dim=40, paths_per_cell=1000, basis=srmc.LP1))}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="one short workload (for ncu)")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--sweep", action="store_true", help="BASELINE config 5: M x N sweep (1 GPU)")
    a = ap.parse_args()
    todo = QUICK if a.quick else WORKLOADS
    if a.sweep:
        todo = {}
        for M in (100, 1000, 10000):
            for N in (10, 20, 50, 100):
                todo[f"c5-sin-d2-lp1-64^2-N{N}-M{M}"] = (lambda: srmc.sin_bench_problem(2),
                                                        dict(steps=N, cells_per_dim=64, paths_per_cell=M))
                todo[f"c5-sin-d6-lp0-8^6-N{N}-M{M}"] = (lambda: srmc.sin_bench_problem(6),
                                                       dict(steps=N, cells_per_dim=8, paths_per_cell=M, basis=srmc.LP0))
    for name, (mk, kw) in todo.items():
        p, c = mk(), srmc.config(**kw)
        srmc.solve(p, c)  # warm-up (module load, allocations)
        best_dev, best_e2e, st = math.inf, math.inf, None
        for _ in range(a.reps):
            t0 = time.perf_counter()
            t = srmc.solve(p, c)
            e2e = time.perf_counter() - t0
            best_dev = min(best_dev, t.stats["device_seconds"])
            best_e2e = min(best_e2e, e2e)
            st = t.stats
        ps = st["path_steps"]
        print(json.dumps({"workload": name, "metric": "path-steps/s (SRMC backward solve)",
                          "value": ps / best_dev, "unit": "path-steps/s", "device_seconds": best_dev,
                          "e2e": {"value": ps / best_e2e, "seconds": best_e2e, "d2h_bytes": t.y.nbytes},
                          "path_steps": ps, "cells": c.cells_per_dim ** p.dim, "kernel_launches": st["kernel_launches"],
                          "dtype": "f64", "data": "synthetic (counter-based Philox on the device)"}), flush=True)


if __name__ == "__main__":
    main()
