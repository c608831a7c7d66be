#!/bin/bash
# tests + smoke + bench of record + ncu launch list (+ full capture of K1/K2) + C4 check
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/r9_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r9_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r9_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r9_smoke.log
timeout 900 python bench.py > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err; echo "bench rc=$?" >> gpurun_out/r9_bench.err
timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r9_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r9_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/r9_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_responses_mma|k_project_mma" -s 30 -c 2 -o gpurun_out/r9_full python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r9_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r9_ncu_full.log
timeout 900 python scratch/c4_check.py > gpurun_out/r9_c4.log 2>&1
