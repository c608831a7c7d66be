#!/bin/bash
# Round-2 refresh after the K2 batch and SRMC Morton changes (run under gpurun): launch list
# of the bench command, ncu --set full of K2 and of the config-4 SRMC step (each command
# first exits 0 without ncu).
set -u
O=gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/p_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/p_bench_ncu.log 2>&1
echo "launches rc=$?"
python tools/k1_run.py --paths 20000000 > $O/p_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_project_mma -s 9 -c 1 -o $O/r02_k2b \
    python tools/k1_run.py --paths 20000000 > $O/p_k2_ncu.log 2>&1
echo "k2 rc=$?"
python tools/srmc_c4_quick.py > $O/p_srmc4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_srmc_step -s 1 -c 1 -o $O/r02_srmc_c4b \
    python tools/srmc_c4_quick.py > $O/p_srmc4_ncu.log 2>&1
echo "srmc c4 rc=$?"
