mkdir -p gpurun_out
for lg in 17 18 19 21; do
  echo "LG_ITEM=$lg"
  MCLAHE_MDICT_LG_ITEM=$lg AB_NO_TESTS=1 AB_CONFIGS=l4d bash tools/ab.sh
done
PROF_CONFIGS="4d l4d" bash tools/round_profile.sh
