#!/bin/bash
# Timing probes of the folded-pair blend (MDICT_PROBE; results are wrong by design,
# only the interp pass time is read), rebuilt on the box.
mkdir -p gpurun_out
export PATH=$PATH:/usr/local/cuda/bin
for pr in ${PROBES:-0 1 2 3 4 5}; do
  touch paper_1906_11355_b200/csrc/k_interp_mdict.cu
  make -s -C paper_1906_11355_b200/csrc -j8 EXTRA=-DMDICT_PROBE=$pr > gpurun_out/probe_build_$pr.log 2>&1 || { echo build $pr failed; tail -5 gpurun_out/probe_build_$pr.log; continue; }
  for c in ${AB_CONFIGS:-4d}; do
    echo "PROBE $pr $c $(timeout 300 python tools/profile_run.py --config $c --iters 2 --time 2>&1 | tail -2 | head -1)"
  done
done
