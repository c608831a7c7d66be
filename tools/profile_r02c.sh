#!/bin/bash
# Final round-2 ncu captures of K1 and K2 on the shipped build (run under gpurun; each
# command first exits 0 without ncu)
O=gpurun_out
python tools/k1_run.py --paths 20000000 > $O/p_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_responses_ws -s 9 -c 1 -o $O/r02_k1c \
    python tools/k1_run.py --paths 20000000 > $O/p_k1_ncu.log 2>&1
echo "k1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_project_mma -s 9 -c 1 -o $O/r02_k2c \
    python tools/k1_run.py --paths 20000000 > $O/p_k2_ncu.log 2>&1
echo "k2 rc=$?"
