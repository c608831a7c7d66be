#!/bin/bash
# ncu launch list of the default bench command (after it exits 0 without ncu)
O=gpurun_out
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/p_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/p_bench_ncu.log 2>&1
echo "launches rc=$?"
