"""Small solve configurations shared by the golden generator and the tests.

Each case is a (ProblemSpec, RunConfig) pair from the reference's own test
and acceptance suites, sized so the CPU oracle finishes in well under a
second: SinBenchmark families (benchmark.cpp:30-67), the driverless /
constant-terminal / linear-terminal problems of proj/tests/test_solver.cpp,
and the truncation-counter problem (test_solver.cpp:291-303).
"""
from __future__ import annotations

from paper_2407_21084_b200 import _abi

TRAIN = 1 << 40  # stream_ids::kStepShift


def sid(step: int, path: int) -> int:
    return (step << 40) | path


DRAW_STREAMS = [("t0_0", sid(0, 0)), ("t1_5", sid(1, 5)), ("t3_2^32+7", sid(3, 2**32 + 7)),
                ("t19_2^39+3", sid(19, 2**39 + 3)), ("eval2_17", (1 << 63) | sid(2, 17)),
                ("raw7", 7)]

CASES = [
    dict(name="sin_d1_full20_q0", problem="sin", dim=1, kind=0, degrees=(20,), steps=5, paths=3000,
         damping=0.0, seed=7),
    dict(name="sin_d2_hyp6_q2.1", problem="sin", dim=2, kind=2, degrees=(6,), steps=5, paths=4000,
         damping=2.1, seed=4242, mse=True),
    dict(name="sin_d2_hyp6_q2.1_recompute", problem="sin", dim=2, kind=2, degrees=(6,), steps=5,
         paths=4000, damping=2.1, seed=4242, memory_mode=1),
    dict(name="sin_d2_total4_mu1_center", problem="sin", dim=2, kind=1, degrees=(4,), steps=4,
         paths=2500, damping=0.0, seed=11, mu=1.0, center=(0.5, -0.25)),
    dict(name="sin_d3_hyp8_q5.1", problem="sin", dim=3, kind=2, degrees=(8,), steps=4, paths=3000,
         damping=5.1, seed=3, mse=True),
    dict(name="sin_d4_hyp16_q5.1", problem="sin", dim=4, kind=2, degrees=(16,), steps=3, paths=2100,
         damping=5.1, seed=5),
    dict(name="sin_d2_full_4x7", problem="sin", dim=2, kind=0, degrees=(4, 7), steps=3, paths=1500,
         damping=0.0, seed=9),
    dict(name="const_terminal_driverless", problem="custom", dim=1, kind=0, degrees=(12,), steps=5,
         paths=400, damping=0.0, seed=17, terminal=_abi.TERMINAL_CONST, terminal_params=(1.0,),
         driver=_abi.DRIVER_ZERO, growth_g=1.0),
    dict(name="truncation_every_value", problem="custom", dim=1, kind=0, degrees=(3,), steps=4, paths=100,
         damping=0.0, seed=8, terminal=_abi.TERMINAL_CONST, terminal_params=(2.0,), driver=_abi.DRIVER_Y,
         growth_g=0.1),
    dict(name="linear_terminal_eta1", problem="custom", dim=1, kind=0, degrees=(10,), steps=4, paths=2000,
         damping=2.1, seed=500, terminal=_abi.TERMINAL_X0, driver=_abi.DRIVER_ZERO, growth_g=1.0,
         growth_exp_g=1.0),
    dict(name="const_driver", problem="custom", dim=1, kind=0, degrees=(6,), steps=4, paths=1000,
         damping=0.0, seed=12, terminal=_abi.TERMINAL_X0, driver=_abi.DRIVER_CONST, driver_params=(0.7,),
         growth_g=1.0, growth_exp_g=1.0, growth_f=0.7),
    dict(name="scalar_diffusion_drift", problem="custom", dim=2, kind=0, degrees=(4, 4), steps=3,
         paths=1500, damping=1.0, seed=21, terminal=_abi.TERMINAL_SIN_SUM, terminal_params=(0.6, 0.5),
         driver=_abi.DRIVER_SIN_BENCH, driver_params=(0.6, 0.5), drift=_abi.DRIFT_CONST,
         drift_params=(0.3,), diffusion=_abi.DIFFUSION_SCALAR, diffusion_params=(0.8,), growth_g=2.6,
         growth_f=1.0, lipschitz_f=2.0),
]

# row f4: general-mu Student measure (Boost students_t restated in include/qrmc_student_t.h,
# used by the reference build's shim too) and per-coordinate drift / diagonal sigma functors
F4_CASES = [
    dict(name="sin_d2_hyp6_mu3.5", problem="sin", dim=2, kind=2, degrees=(6,), steps=4, paths=3000,
         damping=2.1, seed=31, mu=3.5),
    dict(name="sin_d3_total5_mu0.7_center", problem="sin", dim=3, kind=1, degrees=(5,), steps=3, paths=2500,
         damping=2.1, seed=32, mu=0.7, center=(0.3, -0.2, 0.1)),
    dict(name="sin_d4_hyp12_mu6", problem="sin", dim=4, kind=2, degrees=(12,), steps=3, paths=2048,
         damping=5.1, seed=33, mu=6.0),
    dict(name="ou_affine_diag_d3", problem="custom", dim=3, kind=2, degrees=(8,), steps=4, paths=3000,
         damping=2.1, seed=34, terminal=_abi.TERMINAL_SIN_SUM, terminal_params=(0.6, 0.577),
         driver=_abi.DRIVER_SIN_BENCH, driver_params=(0.6, 0.577), drift=_abi.DRIFT_AFFINE,
         drift_vec=(0.1, -0.2, 0.05, 0, 0, 0, 0, 0, -0.5, -0.3, -1.0, 0, 0, 0, 0, 0),
         diffusion=_abi.DIFFUSION_DIAG, diffusion_vec=(0.8, 1.1, 0.6), growth_g=2.6, growth_f=1.0,
         lipschitz_f=2.0),
    dict(name="affine_diag_d2_mu3", problem="custom", dim=2, kind=0, degrees=(5, 5), steps=3, paths=2000,
         damping=0.0, seed=35, mu=3.0, terminal=_abi.TERMINAL_X0, driver=_abi.DRIVER_Y,
         drift=_abi.DRIFT_AFFINE, drift_vec=(0.2, 0.0, 0, 0, 0, 0, 0, 0, 0.1, -0.4, 0, 0, 0, 0, 0, 0),
         diffusion=_abi.DIFFUSION_DIAG, diffusion_vec=(1.3, 0.5), growth_g=1.0, growth_exp_g=1.0,
         growth_f=1.0, lipschitz_f=1.0),
]

PATH_CASES = [
    dict(name="paths_sin_d2", problem="sin", dim=2, kind=2, degrees=(6,), steps=5, paths=10, damping=0.0,
         seed=42, step=1, first=0, n=6),
    dict(name="paths_sin_d3_bigm", problem="sin", dim=3, kind=2, degrees=(4,), steps=4, paths=2**34,
         damping=0.0, seed=99, step=2, first=2**33 + 5, n=3),
    dict(name="paths_mu1_center", problem="sin", dim=2, kind=0, degrees=(3, 3), steps=6, paths=10,
         damping=0.0, seed=5, step=0, first=3, n=4, mu=1.0, center=(1.0, -2.0)),
    dict(name="paths_drift_scalar", problem="custom", dim=2, kind=0, degrees=(2, 2), steps=4, paths=10,
         damping=0.0, seed=6, step=0, first=0, n=4, terminal=_abi.TERMINAL_SIN_SUM, terminal_params=(0.6, 0.5),
         driver=_abi.DRIVER_ZERO, drift=_abi.DRIFT_CONST, drift_params=(0.3,), diffusion=_abi.DIFFUSION_SCALAR,
         diffusion_params=(0.8,)),
]


def build_case(case: dict):
    dim = case["dim"]
    if case["problem"] == "sin":
        prob = _abi.sin_bench_problem(dim, case.get("kappa", 0.6), case.get("lam", 0.0), 1.0)
    else:
        prob = _abi.custom_problem(
            dim, case["terminal"], case["driver"], terminal_params=case.get("terminal_params", ()),
            driver_params=case.get("driver_params", ()), drift=case.get("drift", _abi.DRIFT_ZERO),
            drift_params=case.get("drift_params", ()), diffusion=case.get("diffusion", _abi.DIFFUSION_IDENTITY),
            diffusion_params=case.get("diffusion_params", ()), drift_vec=case.get("drift_vec", ()),
            diffusion_vec=case.get("diffusion_vec", ()), growth_g=case.get("growth_g", 0.0),
            growth_exp_g=case.get("growth_exp_g", 0.0), growth_f=case.get("growth_f", 0.0),
            lipschitz_f=case.get("lipschitz_f", 0.0))
    cfg = _abi.ConfigHolder(steps=case["steps"], paths=case["paths"], damping=case["damping"],
                            seed=case["seed"], memory_mode=case.get("memory_mode", 0), gamma_kind=case["kind"],
                            degrees=list(case["degrees"]), mu=case.get("mu", 2.0),
                            center=list(case["center"]) if case.get("center") else None)
    return prob, cfg
