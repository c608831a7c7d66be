"""Device time of the SRMC plans at BASELINE configs 2, 3 (Bergman, tools/srmc_bench.py's
shape) and 4 (median of 3 after 2 warm-ups):
python tools/srmc_time.py [config2] [config3] [config4]  (QRMC_SRMC_LIB / QRMC_SRMC_MORTON for A/B)."""
import math
import statistics
import sys

sys.path.insert(0, ".")
from bench import SRMC_WORKLOADS  # noqa: E402
from paper_2407_21084_b200 import srmc  # noqa: E402

W = {k: (lambda d=d: srmc.sin_bench_problem(d), kw) for k, (_, d, kw) in SRMC_WORKLOADS.items()}
W["config3"] = (lambda: srmc.bergman_problem(4, 0.05, 0.2, 0.01, 0.06, 100.0, 0.5),
                dict(steps=20, cells_per_dim=24, paths_per_cell=500, basis=1, lo=math.log(100) - 0.6,
                     hi=math.log(100) + 0.6))
for key in sys.argv[1:] or ["config2", "config3", "config4"]:
    mk, kw = W[key]
    p = mk()
    plan = srmc.SrmcPlan(p, srmc.config(**kw), 0, 0, 1, None)
    for _ in range(2):
        plan.run()
    t = statistics.median(plan.run()["device_seconds"] for _ in range(3))
    ps = kw["cells_per_dim"] ** p.dim * kw["paths_per_cell"] * kw["steps"]
    print(f"{key}: {t * 1e3:.1f} ms  {ps / t:.3e} path-steps/s")
    plan.close()
