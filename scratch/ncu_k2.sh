#!/bin/bash
# one ncu --set full capture of the tensor-core K1 (tuning only): $1 = output name
export QRMC_GPU_LIB=${QRMC_GPU_LIB:-$PWD/paper_2407_21084_b200/_lib/variants/libqrmc_gpu_mma4.so}
timeout 300 python bench.py --paths 500000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$1.plain.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_project_mma --launch-skip 10 -c 1 -o gpurun_out/$1 python bench.py --paths 500000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
