#!/bin/bash
# ncu --set full captures of the hot kernels (one launch each) for profiles/:
# 4D (range, histogram, folded-pair dictionary blend), Large 4D (range, histogram,
# folded-pair blend), 5D blend.  PROF_CONFIGS limits the set (default: all).
mkdir -p gpurun_out
CFGS=${PROF_CONFIGS:-"4d l4d 5d"}
for c in $CFGS; do
  case $c in
    4d)  k='regex:k_interp_mdict|k_hist_pencil|k_range_pencil'; n=3 ;;
    l4d) k='regex:k_interp_mdict|k_hist_pencil|k_global_range'; n=3 ;;
    5d)  k='regex:k_interp_pencil|k_hist_pencil'; n=2 ;;
    *)   k="regex:${PROF_KERNELS:-k_}"; n=${PROF_COUNT:-4} ;;
  esac
  ncu --set full --import-source on --clock-control none -k "$k" -c $n \
      -o gpurun_out/prof_$c -f python tools/profile_run.py --config $c --iters 1 > gpurun_out/prof_$c.log 2>&1
  echo "$c rc=$?"
done
