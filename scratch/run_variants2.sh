#!/bin/bash
# parity + small bench of each variant library (tuning only); args: variant names
for n in "$@"; do
  export QRMC_GPU_LIB=$PWD/paper_2407_21084_b200/_lib/variants/libqrmc_gpu_$n.so
  echo "== $n"
  timeout 300 python scratch/mma_check.py 2>&1 | python3 -c "import sys,json; L=[json.loads(l) for l in sys.stdin if l.startswith('{')]; print('maxrelerr', max(d['relerr'] for d in L), 'counters', all(d['apps'][0]==d['apps'][1] and d['clipped'][0]==d['clipped'][1] for d in L))"
  timeout 300 python bench.py --paths 2000000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), {k: round(v,3) for k,v in d['kernel_seconds_per_solve'].items()})"
done
