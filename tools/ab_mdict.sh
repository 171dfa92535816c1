mkdir -p gpurun_out
MCLAHE_MDICT_STG=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo stg_tests_rc=$?; tail -2 gpurun_out/ab_tests.log
for cfg in 4d l4d; do
  for v in 0 1; do
    if [ $v = 1 ]; then export MCLAHE_MDICT_STG=1; else unset MCLAHE_MDICT_STG; fi
    python bench.py --config $cfg --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_${cfg}_$v.json 2>gpurun_out/ab_${cfg}_$v.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_${cfg}_$v.json').read().strip().splitlines()[-1]); p=d['passes']
print('$cfg stg=$v', round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in p.items()})"
  done
done
