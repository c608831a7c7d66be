#!/bin/bash
# per-warp phase clocks of K1 variants (tuning only): args variant names
for n in "$@"; do
  QRMC_GPU_LIB=$PWD/paper_2407_21084_b200/_lib/variants/libqrmc_gpu_$n.so timeout 300 python bench.py --paths 2000000 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/phase_$n.log 2>&1
done
