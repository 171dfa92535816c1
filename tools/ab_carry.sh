export PATH=$PATH:/usr/local/cuda/bin
touch paper_1906_11355_b200/csrc/k_hist.cu
make -s -C paper_1906_11355_b200/csrc -j8 EXTRA=-DK2_PRED_RED_CARRY=1 > gpurun_out/carry_build.log 2>&1 || tail -5 gpurun_out/carry_build.log
ENVS="carry1:MCLAHE_K2_CARRY=1 carry0:MCLAHE_K2_CARRY=0" AB_CONFIGS="4d 5d l4d 3d" bash tools/ab_env.sh
