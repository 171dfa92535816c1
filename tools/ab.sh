#!/bin/bash
# Quick A/B on the GPU box: parity subset + device-only bench lines for the
# configs in AB_CONFIGS (default 4d), passes breakdown on stdout.
mkdir -p gpurun_out
CFGS=${AB_CONFIGS:-4d}
if [ -z "$AB_NO_TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q ${AB_TESTS:+-k "$AB_TESTS"} > gpurun_out/ab_tests.log 2>&1
  echo "tests rc=$? $(tail -1 gpurun_out/ab_tests.log)"
fi
for c in $CFGS; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "FAILED", e); print(open(f"gpurun_out/ab_{c}.err").read()[-2000:]); sys.exit()
p = d.get("passes", {})
print(c, f"{d['value']/1e9:.1f} Gvox/s {d['ms_per_step']:.3f} ms/step", " ".join(f"{k}={v['ms']:.3f}" for k, v in p.items()), "clk", d.get("clocks", {}).get("sm_mhz"))
PY
done
