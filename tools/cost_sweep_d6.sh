for c in "16 10 48" "12 10 48" "12 10 64" "20 10 48" "16 8 48" "16 12 48" "16 10 64" "16 10 32" "16 10 48"; do
  set -- $c
  echo -n "step=$1 nb=$2 epi=$3 "
  QRMC_COST_STEP=$1 QRMC_COST_NB=$2 QRMC_COST_EPI=$3 python tools/k1_run.py --dim 6 --deg 64 --steps 10 2>&1 | tail -1 | cut -c1-75
done
