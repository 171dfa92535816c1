#!/bin/bash
# One-shot measurement set for the docs: default bench (4D, with e2e and CPU
# baseline), the reference arm, every config's device numbers, the ncu
# launch list of the default bench command.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_4d.json 2> gpurun_out/bench_4d.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in 2d 3d l4d 5d; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_4d.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
tail -c 600 gpurun_out/bench_4d.json
