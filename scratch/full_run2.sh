#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full2.json 2> gpurun_out/bench_full2.err; echo "bench rc=$?" >> gpurun_out/bench_full2.err
timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/plain_launch2.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_responses|k_project" -s 30 -c 2 -o gpurun_out/prof_full2 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full2b.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full2b.log
