for ch in 16 24 32; do
  for rep in 1 2; do
  MCLAHE_CHUNKS=$ch python bench.py --config 4d --no-cpu-baseline --e2e-steps 10 --steps 3 > gpurun_out/ch_$ch.json 2>gpurun_out/ch_$ch.err
  python -c "
import json;d=json.loads(open('gpurun_out/ch_$ch.json').read().strip().splitlines()[-1]);e=d['e2e'];print('CHUNKS $ch', round(e['ms_per_step'],3),'ms', round(e['value']/1e9,3),'Gvox/s')"
  done
done
