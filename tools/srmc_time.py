"""Device time of the SRMC plans at BASELINE configs 2 and 4 (median of 3 after 2 warm-ups):
python tools/srmc_time.py [config2] [config4]  (QRMC_SRMC_LIB / QRMC_SRMC_MORTON for A/B)."""
import statistics
import sys

sys.path.insert(0, ".")
from bench import SRMC_WORKLOADS  # noqa: E402
from paper_2407_21084_b200 import srmc  # noqa: E402

for key in sys.argv[1:] or list(SRMC_WORKLOADS):
    name, d, kw = SRMC_WORKLOADS[key]
    plan = srmc.SrmcPlan(srmc.sin_bench_problem(d), srmc.config(**kw), 0, 0, 1, None)
    for _ in range(2):
        plan.run()
    t = statistics.median(plan.run()["device_seconds"] for _ in range(3))
    ps = kw["cells_per_dim"] ** d * kw["paths_per_cell"] * kw["steps"]
    print(f"{key} {name}: {t * 1e3:.1f} ms  {ps / t:.3e} path-steps/s")
    plan.close()
