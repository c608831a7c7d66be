#!/bin/bash
# ncu --set full of the SRMC step kernel at configs 2 and 4 (run under gpurun; each command
# first exits 0 without ncu). Args: output tag.
T=${1:-x}
O=gpurun_out
python tools/srmc_bench.py --quick --reps 1 > $O/p_srmc2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_srmc_step -s 1 -c 1 -o $O/srmc_c2_$T \
    python tools/srmc_bench.py --quick --reps 1 > $O/p_srmc2_ncu.log 2>&1
echo "srmc c2 rc=$?"
python tools/srmc_c4_quick.py > $O/p_srmc4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_srmc_step -s 1 -c 1 -o $O/srmc_c4_$T \
    python tools/srmc_c4_quick.py > $O/p_srmc4_ncu.log 2>&1
echo "srmc c4 rc=$?"
