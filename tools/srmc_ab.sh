# A/B of SRMC build variants at config 4: device time and DRAM bytes per step launch
V=paper_2407_21084_b200/_lib/variants
for v in "QRMC_SRMC_MORTON=1" "QRMC_SRMC_MORTON=0" ${SRMC_AB_VARIANTS}; do
  for m in 0 1; do
  echo "== $v morton=$m"
  env QRMC_SRMC_MORTON=$m $v timeout 300 python tools/srmc_time.py ${SRMC_AB_CONFIGS:-config4}
  env QRMC_SRMC_MORTON=$m $v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_srmc_step -c 2 python tools/srmc_c4_quick.py 2>&1 | grep -E "dram__|gpu__time" | tail -3
  done
done
