#!/bin/bash
# After tools/round_profile.sh on the GPU box: text summaries of the ncu reports
# (what profiles/ keeps), then drop the large reports except the 4D one
# (gpurun_out/ merges back at most 64 MiB).
cd "$(dirname "$0")/.."
S=gpurun_out
python tools/ncu_summary.py $S/prof_4d.ncu-rep k_interp_mdict > $S/ncu_4d_interp_mdict.txt 2>&1
python tools/ncu_summary.py $S/prof_4d.ncu-rep k_hist_pencil > $S/ncu_4d_hist_pencil.txt 2>&1
python tools/ncu_summary.py $S/prof_4d.ncu-rep k_range_pencil > $S/ncu_4d_range_pencil.txt 2>&1
python tools/ncu_summary.py $S/prof_l4d.ncu-rep k_interp_mdict > $S/ncu_l4d_interp.txt 2>&1
python tools/ncu_summary.py $S/prof_l4d.ncu-rep k_hist_pencil > $S/ncu_l4d_hist.txt 2>&1
python tools/ncu_summary.py $S/prof_5d.ncu-rep k_interp_pencil > $S/ncu_5d_interp.txt 2>&1
python tools/ncu_summary.py $S/prof_5d.ncu-rep k_hist_pencil > $S/ncu_5d_hist.txt 2>&1
for c in 4d l4d 5d; do python tools/ncu_stalls.py $S/prof_$c.ncu-rep k_ > $S/ncu_${c}_stalls.txt 2>&1; done
python tools/launch_summary.py $S/launches_4d.csv > $S/launches_4d_summary.txt 2>&1
rm -f $S/prof_l4d.ncu-rep $S/prof_5d.ncu-rep
ls -la $S | head -40
