#!/usr/bin/env python3
"""BASELINE config 1 restated for GQRMDP: d=2, full index set
Gamma_F(31,31) (#Gamma=1024), q=0, N=10, M=102,400, SinBenchmark -- the reference's own
CPU-runnable case (1.639 s on the survey container's 8 cores).

    python tools/config1_run.py [--out profiles/r02_config1.json]

Times the device solve (plan, CUDA events, median of 3 after a warm-up) and the public
one-shot call (host buffers, e2e), then the reference build (oracle/_ref, all host cores,
median of 3) on the same inputs, and reports the largest coefficient difference."""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2407_21084_b200 import _abi, api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--paths", type=int, default=102_400)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--out", default=None)
ap.add_argument("--no-ref", action="store_true")
args = ap.parse_args()

L = _abi.lib()
prob = _abi.sin_bench_problem(2)
cfg = _abi.ConfigHolder(steps=args.steps, paths=args.paths, damping=0.0, seed=42, gamma_kind=0, degrees=[31, 31])
plan = C.c_void_p()
err = C.create_string_buffer(1024)
api.raise_for(L.qrmc_gpu_plan_create(None, C.byref(prob), cfg.ref(), C.byref(plan), err, 1024), err.value.decode())
st = _abi.Stats()
dev = []
for r in range(4):
    api.raise_for(L.qrmc_gpu_plan_run(plan, C.byref(st), err, 1024), err.value.decode(), st.error_step)
    if r:
        dev.append(st.device_seconds)
names = [L.qrmc_gpu_plan_kernel_name(plan, w).decode() for w in range(3)]
ks = (C.c_double * 3)()
L.qrmc_gpu_plan_kernel_seconds(plan, ks, None, err, 1024)
K = L.qrmc_gpu_plan_basis_size(plan)
L.qrmc_gpu_plan_destroy(plan)
e2e = []
for _ in range(3):
    t0 = time.perf_counter()
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    e2e.append(time.perf_counter() - t0)
out = {"workload": "config1-gqrmdp: d=2 Gamma_F(31,31) q=0 N=10 M=102400 SinBenchmark", "basis_size": K,
       "kernels": dict(zip(names, ks[:])), "device_seconds_median": statistics.median(dev),
       "e2e_seconds_median": statistics.median(e2e), "reference_survey_8core_s": 1.639}
if not args.no_ref:
    import oracles  # test infrastructure: the reference build as the CPU baseline and checker
    R = oracles.ref() if oracles.have_ref() else oracles.port()
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        ref, rstats = R.backward_solve(prob, cfg, K)
        times.append(time.perf_counter() - t0)
    out["reference_host_seconds_median"] = statistics.median(times)
    out["reference_kind"] = "reference" if oracles.have_ref() else "port"
    out["host_threads"] = min(os.cpu_count() or 1, 256, -(-args.paths // 1024))
    out["max_abs_coeff_diff"] = float(np.abs(coeffs - ref).max())
    out["max_abs_coeff"] = float(np.abs(ref).max())
    out["speedup_device_vs_host_ref"] = out["reference_host_seconds_median"] / out["device_seconds_median"]
    out["speedup_e2e_vs_host_ref"] = out["reference_host_seconds_median"] / out["e2e_seconds_median"]
print(json.dumps(out))
if args.out:
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")
