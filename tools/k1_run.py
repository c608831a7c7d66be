#!/usr/bin/env python3
"""One prepared backward solve of the bench workload (tools for ncu captures).

    python tools/k1_run.py [--paths M] [--runs R] [--dim 4 --deg 100 --steps 20]

Prints per-kernel device seconds of the last run; QRMC_K1 / QRMC_K2 select kernel families."""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_21084_b200 import _abi, api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--paths", type=int, default=2_000_000)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--dim", type=int, default=4)
ap.add_argument("--deg", type=int, default=100)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--damping", type=float, default=5.1)
args = ap.parse_args()
L = _abi.lib()
prob = _abi.sin_bench_problem(args.dim)
cfg = _abi.ConfigHolder(steps=args.steps, paths=args.paths, damping=args.damping, seed=42, gamma_kind=2,
                        degrees=[args.deg])
plan = C.c_void_p()
err = C.create_string_buffer(1024)
api.raise_for(L.qrmc_gpu_plan_create(None, C.byref(prob), cfg.ref(), C.byref(plan), err, 1024), err.value.decode())
st = _abi.Stats()
ks = (C.c_double * 3)()
for r in range(args.runs):
    api.raise_for(L.qrmc_gpu_plan_run(plan, C.byref(st), err, 1024), err.value.decode(), st.error_step)
    L.qrmc_gpu_plan_kernel_seconds(plan, ks, None, err, 1024)
    if args.runs > 1:
        print(json.dumps({"run": r, "kernel_seconds": ks[:]}), flush=True)
K = L.qrmc_gpu_plan_basis_size(plan)
n, m = args.steps, args.paths
names = [L.qrmc_gpu_plan_kernel_name(plan, w).decode() for w in range(3)]
k1_flops = 2.0 * K * m * n * (n - 1) / 2.0
print(json.dumps({"kernels": dict(zip(names, ks[:])), "device_s": st.device_seconds,
                  "k1_tflops": k1_flops / ks[0] / 1e12, "k1_frac": k1_flops / ks[0] / 1e12 / 37.1,
                  "path_steps_per_s": m * n * (n + 1) / 2 / st.device_seconds}))
L.qrmc_gpu_plan_destroy(plan)
