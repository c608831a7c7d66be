# d=4 parity of the tensor-core K1 against the oracle port + the series K1 (tuning only).
import sys, time, json, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracles
from paper_2407_21084_b200 import _abi, api
P = oracles.port()
for (kind, deg, N, M, q) in [(2, [16], 6, 20000, 5.1), (2, [100], 3, 4096, 5.1), (1, [6], 4, 8192, 5.1), (0, [3], 4, 8192, 5.1)]:
    prob = _abi.sin_bench_problem(4)
    cfg = _abi.ConfigHolder(steps=N, paths=M, damping=q, seed=42, gamma_kind=kind, degrees=deg)
    K = len(P.gamma(kind, 4, deg)[0])
    t = time.time(); a, sa = P.backward_solve(prob, cfg, K); tr = time.time() - t
    b, sb, _ = api.backward_solve(prob, cfg)
    err = float(np.abs(a - b).max() / max(1.0, np.abs(a).max()))
    print(json.dumps(dict(kind=kind, deg=deg, K=K, relerr=err, apps=[int(sa.applications), int(sb.applications)],
                          clipped=[int(sa.clipped), int(sb.clipped)], t_port=tr, dev=sb.device_seconds)), flush=True)
