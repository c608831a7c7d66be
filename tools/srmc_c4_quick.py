"""Two steps of BASELINE config 4 (d=6, LP0, 16^6 hypercubes, M=100) -- the ncu target for the sub-warp SRMC kernel."""
import sys; sys.path.insert(0, '.')
from paper_2407_21084_b200 import srmc
p = srmc.sin_bench_problem(6)
c = srmc.config(2, 16, 100, basis=srmc.LP0)
srmc.solve(p, c)
