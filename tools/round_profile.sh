#!/bin/bash
# ncu --set full captures of the hot kernels (one launch each) for profiles/:
# 4D (range, histogram, folded-pair dictionary blend), Large 4D (range, histogram,
# folded-pair blend), 5D blend.
mkdir -p gpurun_out
ncu --set full --import-source on -k regex:"k_interp_mdict|k_hist_pencil|k_range_pencil" -c 3 \
    -o gpurun_out/prof_4d -f python tools/profile_run.py --config 4d --iters 1 > gpurun_out/prof_4d.log 2>&1
ncu --set full --import-source on -k regex:"k_interp_mdict|k_hist_pencil|k_global_range" -c 3 \
    -o gpurun_out/prof_l4d -f python tools/profile_run.py --config l4d --iters 1 > gpurun_out/prof_l4d.log 2>&1
ncu --set full --import-source on -k regex:"k_interp_pencil" -c 2 \
    -o gpurun_out/prof_5d -f python tools/profile_run.py --config 5d --iters 1 > gpurun_out/prof_5d.log 2>&1
