#!/bin/bash
# parity + M=2e6 bench of a K1 variant library (tuning only)
export QRMC_GPU_LIB=${QRMC_GPU_LIB:-$PWD/paper_2407_21084_b200/_lib/variants/libqrmc_gpu_mma4.so}
timeout 300 python scratch/mma_check.py 2>&1 | tail -8
timeout 300 python bench.py --paths 2000000 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_seconds_per_solve'])"
