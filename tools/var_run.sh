# timing experiments (tools/build_variants.py): K1 seconds per solve at M = 2e6
for v in "$@"; do
  echo -n "$v "; QRMC_GPU_LIB=paper_2407_21084_b200/_lib/variants/libqrmc_gpu_$v.so python tools/k1_run.py 2>&1 | tail -1 | cut -c1-60
done
