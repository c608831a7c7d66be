#!/bin/bash
# one ncu --set full capture of K1 at M = 2e6 (cloud step i=10), for shared-memory conflict checks
O=gpurun_out
python tools/k1_run.py > $O/p_k1q.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_responses_ws -s 9 -c 1 -o $O/${1:-k1q} \
    python tools/k1_run.py > $O/p_k1q_ncu.log 2>&1
echo "rc=$?"
