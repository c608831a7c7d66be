# print the K1 tensor-core unit layout of the bench workload (tuning only; needs a GPU)
import sys; sys.path.insert(0, ".")
from paper_2407_21084_b200 import _abi, api
prob = _abi.sin_bench_problem(4)
cfg = _abi.ConfigHolder(steps=20, paths=40960, damping=5.1, seed=42, gamma_kind=2, degrees=[100])
api.backward_solve(prob, cfg)
