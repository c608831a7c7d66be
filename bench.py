#!/usr/bin/env python3
"""Benchmark: full GQRMDP backward solve on B200 (path-steps/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" of this benchmark is one full backward solve (qrmc::backward_solve,
proj/src/solver.cpp:109-226) of the BASELINE.json configs[1] workload as
restated in SURVEY.md 8(d): SinBenchmark d=4 (kappa 0.6, lambda 1/2, T=1),
hyperbolic index set Gamma_H(4,100) (#Gamma = 12,752), damping q = 5.1,
N = 20 time steps, M = 2e7 paths per GPU per backward step (weak scaling),
Student mu=2 sampling measure, training seed 42, store-cloud mode.

Metric: simulated path-steps per second = M N (N+1)/2 / solve time
(SURVEY.md 8(d)); `value` is device-timed (CUDA events on the solver's
stream, inputs resident), `e2e` goes through the public C ABI call
qrmc_gpu_backward_solve with host buffers. With --impl reference the same
metric is measured for the reference's own CPU solver (oracle/_ref, the
unmodified reference sources) on a bounded sample of M on all host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

WORKLOAD = dict(name="sinbench-d4-hyperbolic100-q5.1-N20", dim=4, kappa=0.6, lam=0.0, horizon=1.0,
                gamma_kind="hyperbolic", degrees=(100,), damping=5.1, steps=20, mu=2.0, seed=42)
# BASELINE config 4 restated for GQRMDP: d=6, Gamma_H(6,64) (K=76,433), N=10,
# M = 2e7 per GPU -- a second line in the JSON (`gqrmdp_config4`), one timed solve
WORKLOAD_C4 = dict(WORKLOAD, name="sinbench-d6-hyperbolic64-q5.1-N10", dim=6, degrees=(64,), steps=10)
DEFAULT_PATHS_PER_GPU = 20_000_000
CPU_SAMPLE_PATHS = 16_384  # 16 lanes of 1024 paths: saturates 16 host cores (parallel.hpp:21-22)
METRIC = "simulated paths x time-steps per second per full backward solve"
UNIT = "path-steps/s"


def traffic_per_launch(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    --set full capture of this workload (profiles/roofline_traffic.json), or None."""
    f = ROOT / "profiles" / "roofline_traffic.json"
    if not f.exists():
        return None
    try:
        return json.loads(f.read_text())[kernel]["dram_bytes_per_launch"]
    except (KeyError, ValueError):
        return None


def peaks() -> dict:
    p = {}
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        p.update(json.loads(f.read_text()))
    # FP64 peak measured on this pool's B200 (profiles/r01_fp64_peak.txt: DMMA m8n8k4
    # 37.1 TF/s, DFMA 34.2 TF/s, cuBLAS DGEMM 35.5 TF/s). MEASURED_PEAKS.json has no FP64 entry.
    p.setdefault("fp64_tflops", 37.1)
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def path_steps(m: int, n: int) -> int:
    return m * n * (n + 1) // 2


def flops_alg(k: int, m: int, n: int) -> float:
    # 2 FLOPs (one FMA) per basis term per path-step
    return float(k) * m * n * (n + 1)


def make_problem_config(paths: int, w: dict | None = None):
    from paper_2407_21084_b200 import _abi
    w = w or WORKLOAD
    prob = _abi.sin_bench_problem(w["dim"], w["kappa"], w["lam"], w["horizon"])
    cfg = _abi.ConfigHolder(steps=w["steps"], paths=paths, damping=w["damping"], seed=w["seed"],
                            gamma_kind=_abi.GAMMA_KINDS[w["gamma_kind"]], degrees=w["degrees"], mu=w["mu"])
    return prob, cfg


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU, NCCL) on this
    node with the same arguments, as the driver's own torchrun launch would."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------ reference CPU
def cpu_reference_solve(paths: int) -> tuple[float, str]:
    """Wall time of the reference's own backward_solve (oracle/_ref: the unmodified
    reference sources, proj/src/solver.cpp:109-226) on all host cores. Nothing of this
    repo's CUDA library is loaded on this path: #Gamma comes from the reference's own
    MultiIndexSet (multi_index.cpp:96-173)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles  # test infrastructure: the reference build, only for the baseline leg
    from paper_2407_21084_b200 import _abi  # ctypes structs only (no library load)
    R = oracles.ref() if oracles.have_ref() else None
    kind = "reference"
    if R is None:
        R = oracles.port()
        kind = "port"
    prob, cfg = make_problem_config(paths)
    k = int(R.gamma(cfg.c.gamma_kind, prob.dim, list(WORKLOAD["degrees"]))[0].shape[0])
    t0 = time.perf_counter()
    R.backward_solve(prob, cfg, k)
    return time.perf_counter() - t0, kind


def cpu_baseline_sample(paths: int, repeats: int) -> dict:
    """The reference CPU solver on a bounded sample of the workload: the median of
    `repeats` full N=20 solves at M = paths, and one solve at 2M to show that time is
    linear in M (work and memory are exactly proportional to M), so the
    per-path-step rate extrapolates to the GPU's M."""
    n = WORKLOAD["steps"]
    times, kind = [], "reference"
    for _ in range(repeats):
        t, kind = cpu_reference_solve(paths)
        times.append(t)
    med = statistics.median(times)
    t2, _ = cpu_reference_solve(2 * paths)
    cores = os.cpu_count() or 1
    threads = min(cores, 256, -(-paths // 1024))
    return {"value": path_steps(paths, n) / med, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"median of {repeats} full N={n} backward solves at M={paths} ({med:.1f} s each) on "
                      f"{threads} of {cores} host threads; one solve at M={2 * paths} took {t2:.1f} s "
                      f"(ratio {t2 / med:.2f} vs 2.00 for exact linearity); extrapolated linearly in M "
                      f"to the GPU workload",
            "seconds": times, "linearity_2m_over_m": t2 / med, "extrapolated": True}


def run_reference_arm(args) -> int:
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    n = WORKLOAD["steps"]
    paths = args.cpu_paths
    cores = os.cpu_count() or 1
    threads = min(cores, 256, -(-paths // 1024))
    for _ in range(args.warmup):
        cpu_reference_solve(paths)
    times = []
    kind = "reference"
    for _ in range(args.steps):
        t, kind = cpu_reference_solve(paths)
        times.append(t)
    med = statistics.median(times)
    value = path_steps(paths, n) / med
    t2, _ = cpu_reference_solve(2 * paths)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": med * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD["name"], "paths_per_step_sample": paths, "N": n,
                   "basis": "hyperbolic(4,100) #Gamma=12752", "parallelism": "host threads (lane pool)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"full N={n} backward solve at M={paths} per step, median of {args.steps}; "
                                   f"one solve at M={2 * paths}: {t2:.1f} s vs {med:.1f} s (linear in M); "
                                   f"rate extrapolated linearly to the GPU's M",
                         "linearity_2m_over_m": t2 / med, "extrapolated": True},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ SRMC (row f3)
# The north_star's stratified regression Monte Carlo solver at the literal BASELINE.json
# configs 2 and 4, and config 3 (Bergman) at tools/srmc_bench.py's shape
# (include/qrmc_srmc.h; no reference arm: the reference has no SRMC).
# Hypercubes are partitioned over the ranks and every step's table is all-gathered
# (strong scaling: the cell count is the config's, whatever N).
SRMC_WORKLOADS = {
    "config2": ("sin-d4-lp1-40^4-N20-M1000", 4, dict(steps=20, cells_per_dim=40, paths_per_cell=1000, basis=1)),
    "config4": ("sin-d6-lp0-16^6-N10-M100", 6, dict(steps=10, cells_per_dim=16, paths_per_cell=100, basis=0)),
}
# BASELINE config 3 (Bergman borrowing/lending, d=4, LP1, N=20; the hypercubes and paths
# are this repo's choice, tools/srmc_bench.py): a z-dependent driver, so two passes per step
SRMC_BERGMAN = ("bergman-d4-lp1-24^4-N20-M500", 4,
                dict(steps=20, cells_per_dim=24, paths_per_cell=500, basis=1, lo=math.log(100) - 0.6,
                     hi=math.log(100) + 0.6))
DFMA_PEAK_TFLOPS = 34.2  # builder-measured scalar DFMA peak (profiles/r01_fp64_peak.txt); SRMC runs no tensor op


def srmc_flops_per_path_step(d: int, P: int) -> int:
    """Floating-point operations the SRMC scheme performs per path-step (one cell path, one
    Euler step), counted from its specification (include/qrmc_srmc.h, oracle/srmc_oracle.c):
    start point 3d + basis 2d; d AS241 normal quantiles at 35 each (two degree-7 rational
    polynomials = 28 FMA-flops, division, log, sqrt, scaling); Euler 3d + 1d (sqrt(dt) z);
    projection + cell + local coordinates 7d; local polynomial 2P; SinBenchmark driver
    d + 7 (sin counted once); truncation 0; normal equations P(P+1) (packed Gram, FMA) and
    right-hand side 2 + 2P. RNG integer work is not counted."""
    return 5 * d + 35 * d + 4 * d + 7 * d + 2 * P + (d + 7) + P * (P + 1) + 2 + 2 * P


def srmc_bergman_flops_per_path_step(d: int, P: int) -> int:
    """The Bergman scheme per path-step, counted the same way: two passes over the same
    draws (include/qrmc_srmc.h). Pass 1: path (start 5d, quantiles 35d, Euler 4d, cell 7d),
    next-step polynomial 2P, Gram P(P+1), Z right-hand side d (2 + 2P). Pass 2: the path
    again (51d + 2P), Z_hat at the start d * 2P, driver 3d + 12 (sum of z, borrow/lend
    rates), Y right-hand side 2 + 2P."""
    path = 5 * d + 35 * d + 4 * d + 7 * d + 2 * P
    return (path + P * (P + 1) + d * (2 + 2 * P)) + (path + d * 2 * P + 3 * d + 12 + 2 + 2 * P)


def run_srmc(args, world: int, rank: int, local: int, dist) -> dict:
    import torch
    from paper_2407_21084_b200 import srmc
    out = {}
    todo = {k: (name, d, kw, srmc.sin_bench_problem(d), srmc_flops_per_path_step)
            for k, (name, d, kw) in SRMC_WORKLOADS.items()}
    bname, bd, bkw = SRMC_BERGMAN
    todo["config3"] = (bname, bd, bkw, srmc.bergman_problem(bd, 0.05, 0.2, 0.01, 0.06, 100.0, 0.5),
                       srmc_bergman_flops_per_path_step)
    for key in ("config2", "config3", "config4"):
        name, d, kw, p, flops_fn = todo[key]
        c = srmc.config(**kw)
        nid = None
        if world > 1:
            obj = [srmc.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        plan = srmc.SrmcPlan(p, c, local, rank, world, nid)
        for _ in range(args.srmc_warmup):
            plan.run()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        dev = []
        with ClockSampler(local) as clocks:
            for _ in range(args.srmc_steps):
                dev.append(plan.run()["device_seconds"])
        t = statistics.median(dev)
        if dist is not None:
            tt = torch.tensor([t], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        plan.close()
        cells = kw["cells_per_dim"] ** d
        ps = cells * kw["paths_per_cell"] * kw["steps"]  # whole job (all ranks)
        P = d + 1 if kw["basis"] == 1 else 1
        fl = flops_fn(d, P)
        entry = {"workload": name, "value": ps / t, "unit": "path-steps/s", "seconds_per_solve": t,
                 "cells": cells, "paths_per_cell": kw["paths_per_cell"], "N": kw["steps"], "basis": f"LP{kw['basis']}",
                 "path_passes": 2 if key == "config3" else 1,  # a path-step counts once either way
                 "n_gpus": world, "scaling": "strong (fixed hypercubes, partitioned over the ranks)",
                 "exchange": "ncclAllGather of every step's y table" if world > 1 else "none (1 rank)",
                 "clocks": clocks.summary(),
                 "roofline": {"bound": "fp64", "flops_per_path_step": fl,
                              "achieved": ps * fl / t / 1e12 / world, "peak": DFMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": ps * fl / t / 1e12 / world / DFMA_PEAK_TFLOPS,
                              "peak_source": "of builder-measured scalar DFMA 34.2 TF/s (profiles/r01_fp64_peak.txt)",
                              "note": "per GPU; path generation (Philox, AS241 quantiles) dominates; HBM traffic "
                                      "per path-step is ~2P*8/M bytes (table read + write), far below the ridge"}}
        if world == 1:
            # e2e: the public one-shot call with host tables (allocation, solve, D2H of every
            # step's table), one untimed call first (first-touch of the host pages), then the
            # median of 2
            srmc.solve(p, c)
            e2es = []
            for _ in range(2):
                t0 = time.perf_counter()
                tab = srmc.solve(p, c)
                e2es.append(time.perf_counter() - t0)
            e2e = statistics.median(e2es)
            entry["e2e"] = {"value": ps / e2e, "unit": "path-steps/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": int(tab.y.nbytes)}
            del tab
        out[key] = entry
    return out


def run_gqrmdp_config4(args, L, session, world: int, dist) -> dict:
    """BASELINE config 4 restated for GQRMDP on the same session: one warm-up and one timed
    solve (device time, max over ranks), per-kernel seconds and the dominant kernel's FP64
    fraction (the same algorithmic count as the headline: 2 K FLOPs per evaluation)."""
    import torch
    from paper_2407_21084_b200 import api
    err = C.create_string_buffer(1024)
    m = args.paths
    n = WORKLOAD_C4["steps"]
    prob, cfg = make_problem_config(m * world, WORKLOAD_C4)
    plan = C.c_void_p()
    api.raise_for(L.qrmc_gpu_plan_create(session, C.byref(prob), cfg.ref(), C.byref(plan), err, 1024),
                  err.value.decode())
    stats = _abi_stats()
    try:
        times, ks = [], (C.c_double * 3)()
        for _ in range(2):  # warm-up, timed
            if dist is not None:
                dist.barrier()
            api.raise_for(L.qrmc_gpu_plan_run(plan, C.byref(stats), err, 1024), err.value.decode(), stats.error_step)
            times.append(stats.device_seconds)
        t = times[-1]
        L.qrmc_gpu_plan_kernel_seconds(plan, ks, None, err, 1024)
        if dist is not None:
            tt = torch.tensor([t], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        K = int(L.qrmc_gpu_plan_basis_size(plan))
        names = [L.qrmc_gpu_plan_kernel_name(plan, w).decode() for w in range(3)]
    finally:
        L.qrmc_gpu_plan_destroy(plan)
    k1 = 2.0 * K * m * n * (n - 1) / 2.0 / ks[0] / 1e12
    return {"workload": WORKLOAD_C4["name"], "value": path_steps(m * world, n) / t, "unit": UNIT,
            "seconds_per_solve": t, "basis_size": K, "N": n, "paths_per_gpu": m, "n_gpus": world,
            "kernel_seconds_per_solve": dict(zip(names, ks[:])),
            "roofline": {"kernel": names[0], "bound": "fp64", "achieved": k1, "peak": peaks()["fp64_tflops"],
                         "unit": "TFLOP/s", "frac": k1 / peaks()["fp64_tflops"],
                         "peak_source": "of builder-measured 37.1 TF/s FP64 (profiles/r01_fp64_peak.txt)"},
            "timing": "one solve after one warm-up (device time, CUDA events)"}


def _abi_stats():
    from paper_2407_21084_b200 import _abi
    return _abi.Stats()


# ------------------------------------------------------------------ our arm
def run_ours(args) -> int:
    from paper_2407_21084_b200 import _abi, api
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    import torch
    torch.cuda.set_device(local)
    L = _abi.lib()
    err = C.create_string_buffer(1024)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = (C.c_char * 128)()
        if rank == 0:
            api.raise_for(L.qrmc_gpu_nccl_unique_id(uid, err, 1024), err.value.decode())
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        C.memmove(uid, obj[0], 128)
        uid_ptr = C.cast(uid, C.c_void_p)
    else:
        uid_ptr = None
    session = C.c_void_p()
    api.raise_for(L.qrmc_gpu_session_create(local, rank, world, uid_ptr, C.byref(session), err, 1024),
                  err.value.decode())

    paths_total = args.paths * world  # weak scaling: M per GPU fixed
    n = WORKLOAD["steps"]
    prob, cfg = make_problem_config(paths_total)
    plan = C.c_void_p()
    api.raise_for(L.qrmc_gpu_plan_create(session, C.byref(prob), cfg.ref(), C.byref(plan), err, 1024),
                  err.value.decode())
    K = int(L.qrmc_gpu_plan_basis_size(plan))
    stream = torch.cuda.ExternalStream(L.qrmc_gpu_plan_stream(plan))
    stats = _abi.Stats()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def run_once():
        api.raise_for(L.qrmc_gpu_plan_run(plan, C.byref(stats), err, 1024), err.value.decode(), stats.error_step)

    for _ in range(args.warmup):
        run_once()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernel_s = np.zeros(3)
    ks = (C.c_double * 3)()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            run_once()
            api.raise_for(L.qrmc_gpu_plan_kernel_seconds(plan, ks, None, err, 1024), err.value.decode())
            kernel_s += np.array(ks[:])
        ev1.record(stream)
        barrier()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    if dist is not None:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    per_solve = elapsed / args.steps
    value = path_steps(paths_total, n) / per_solve
    launches = int(stats.kernel_launches) * args.steps

    # roofline of the dominant kernel, phase 1 (k_responses_mma on the FP64 tensor cores
    # for this workload): 2 FLOPs per basis term per future-point evaluation,
    # M_local * sum_i (N-1-i) evaluations per solve, against the measured DMMA peak.
    m_local = args.paths
    resp_flops = 2.0 * K * m_local * n * (n - 1) / 2.0
    resp_s = kernel_s[0] / args.steps
    pk = peaks()
    achieved = resp_flops / resp_s / 1e12
    solve_tflops = flops_alg(K, m_local, n) / per_solve / 1e12

    # e2e: the public C ABI call with host buffers (plan build + H2D, graph, solve, D2H)
    h2d, d2h = C.c_uint64(), C.c_uint64()
    L.qrmc_gpu_plan_io_bytes(plan, C.byref(h2d), C.byref(d2h))
    coeffs = np.zeros((n, K))
    e2e_times = []
    for _ in range(args.e2e_steps):
        barrier()
        t0 = time.perf_counter()
        st = L.qrmc_gpu_backward_solve(session, C.byref(prob), cfg.ref(),
                                       coeffs.ctypes.data_as(C.POINTER(C.c_double)), coeffs.size, None,
                                       C.byref(stats), err, 1024)
        api.raise_for(st, err.value.decode(), stats.error_step)
        barrier()
        e2e_times.append(time.perf_counter() - t0)
    e2e_t = statistics.median(e2e_times)
    if dist is not None:
        t = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    names = [L.qrmc_gpu_plan_kernel_name(plan, w).decode() for w in range(3)]
    L.qrmc_gpu_plan_destroy(plan)

    c4_line = None if args.no_config4 else run_gqrmdp_config4(args, L, session, world, dist)
    srmc_line = None if args.no_srmc else run_srmc(args, world, rank, local, dist)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args.cpu_paths, args.cpu_repeats)
    if dist is not None:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_solve * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD["name"], "d": WORKLOAD["dim"], "basis": "hyperbolic(4,100)",
                       "basis_size": K, "N": n, "paths_per_gpu": args.paths, "paths_total": paths_total,
                       "damping": WORKLOAD["damping"], "seed": WORKLOAD["seed"],
                       "parallelism": f"paths sharded by lane over {world} GPU(s)",
                       "l2": "working set (cloud + responses, 0.8 GB/GPU) larger than L2"},
            "time_to_solution_s": per_solve,
            "fp64_solve_tflops": solve_tflops,
            "fp64_solve_frac": solve_tflops / pk["fp64_tflops"],
            "kernel_seconds_per_solve": {names[0]: kernel_s[0] / args.steps,
                                         names[1]: kernel_s[1] / args.steps,
                                         names[2]: kernel_s[2] / args.steps},
            "roofline": {"kernel": names[0], "bound": "fp64", "achieved": achieved,
                         "peak": pk["fp64_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["fp64_tflops"],
                         "traffic": traffic_per_launch(names[0]),
                         "peak_source": "of builder-measured 37.1 TF/s FP64 (DMMA m8n8k4 microbenchmark on this "
                                        "pool's B200, profiles/r01_fp64_peak.txt; cuBLAS DGEMM 35.5); "
                                        "MEASURED_PEAKS.json has no FP64 entry"},
            "e2e": {"value": path_steps(paths_total, n) / e2e_t, "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d.value), "d2h_bytes_per_step": int(d2h.value)},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if c4_line is not None:
            line["gqrmdp_config4"] = c4_line
        if srmc_line is not None:
            line["srmc"] = srmc_line
        print(json.dumps(line), flush=True)
    L.qrmc_gpu_session_destroy(session)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--paths", type=int, default=DEFAULT_PATHS_PER_GPU, help="paths per GPU per backward step")
    ap.add_argument("--cpu-paths", type=int, default=CPU_SAMPLE_PATHS)
    ap.add_argument("--cpu-repeats", type=int, default=3)
    ap.add_argument("--no-srmc", action="store_true", help="skip the SRMC (row f3) section")
    ap.add_argument("--no-config4", action="store_true", help="skip the GQRMDP config-4 restatement")
    ap.add_argument("--srmc-steps", type=int, default=3)
    ap.add_argument("--srmc-warmup", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
