#!/bin/bash
# C4-shape timing of variant libraries (tuning only)
for n in "$@"; do
  echo "== $n"
  QRMC_GPU_LIB=$PWD/paper_2407_21084_b200/_lib/variants/libqrmc_gpu_$n.so timeout 600 python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2407_21084_b200 import _abi, api
prob = _abi.sin_bench_problem(6)
cfg = _abi.ConfigHolder(steps=10, paths=2_000_000, damping=5.1, seed=42, gamma_kind=2, degrees=[64])
api.backward_solve(prob, cfg)
c, s, w = api.backward_solve(prob, cfg)
L = _abi.lib()
import ctypes as C, numpy as np
print("device_s", round(s.device_seconds, 3))
PY
done
