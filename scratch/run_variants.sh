#!/bin/bash
# Small-bench each K1 shape variant (tuning only).
for so in paper_2407_21084_b200/_lib/variants/*.so; do
  n=$(basename $so .so)
  QRMC_GPU_LIB=$PWD/$so timeout 300 python bench.py --paths 2000000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/var_$n.json 2> gpurun_out/var_$n.err
  echo "$n rc=$?" >> gpurun_out/variants.log
done
