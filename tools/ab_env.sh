#!/bin/bash
# env-knob A/B (no rebuild): ENVS="name:VAR=val,VAR2=val ..." 
mkdir -p gpurun_out
for e in ${ENVS}; do
  name=${e%%:*}; kv=${e#*:}
  (
  IFS=,; for x in $kv; do [ "$x" != "none" ] && export "$x"; done; unset IFS
  for c in ${AB_CONFIGS:-4d}; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/env_${name}_$c.json 2> gpurun_out/env_${name}_$c.err || { echo "ENV $name $c failed"; tail -3 gpurun_out/env_${name}_$c.err; continue; }
    python - "$c" "$name" <<'PY'
import json, sys
c, name = sys.argv[1:3]
d = json.loads(open(f"gpurun_out/env_{name}_{c}.json").read().strip().splitlines()[-1])
p = d.get("passes", {})
print("ENV", name, c, f"{d['value']/1e9:.1f} Gvox/s {d['ms_per_step']:.4f} ms/step", " ".join(f"{k}={v['ms']:.4f}" for k, v in p.items()))
PY
  done
  )
done
