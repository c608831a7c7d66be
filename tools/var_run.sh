# timing experiments (tools/build_variants.py): kernel seconds per solve at M = 2e6 (args: variant names)
for v in "$@"; do
  echo -n "$v "; QRMC_GPU_LIB=paper_2407_21084_b200/_lib/variants/libqrmc_gpu_$v.so python tools/k1_run.py 2>&1 | tail -1 | cut -c1-130
done
