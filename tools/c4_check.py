# C4-shaped check (d=6, hyperbolic(6,64), K=76,433): parity vs the oracle port at small M,
# then device time at M=2e6, N=10 for both kernel families (tuning only).
import sys, time, json, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracles
from paper_2407_21084_b200 import _abi, api
P = oracles.port()
prob = _abi.sin_bench_problem(6)
cfg = _abi.ConfigHolder(steps=3, paths=4096, damping=5.1, seed=42, gamma_kind=2, degrees=[64])
K = len(P.gamma(2, 6, [64])[0])
t = time.time(); a, sa = P.backward_solve(prob, cfg, K); tp = time.time() - t
b, sb, _ = api.backward_solve(prob, cfg)
print(json.dumps(dict(K=K, relerr=float(np.abs(a - b).max() / max(1, np.abs(a).max())), apps=[sa.applications, sb.applications],
                      clipped=[sa.clipped, sb.clipped], t_port=tp)), flush=True)
for fam in ("mma", "series"):
    if fam == "series":
        os.environ["QRMC_K1"] = "series"; os.environ["QRMC_K2"] = "series"
    cfg = _abi.ConfigHolder(steps=10, paths=2_000_000, damping=5.1, seed=42, gamma_kind=2, degrees=[64])
    api.backward_solve(prob, cfg)
    c, s, _ = api.backward_solve(prob, cfg)
    n = 10
    print(fam, json.dumps(dict(device_s=s.device_seconds, path_steps_per_s=2e6 * n * (n + 1) / 2 / s.device_seconds,
                               tflops=2 * K * 2e6 * n * (n + 1) / s.device_seconds / 1e12)), flush=True)
