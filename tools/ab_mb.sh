#!/bin/bash
# A/B: table-build batch of the folded-pair blend (MDICT_BUILD_BATCH), rebuilt on the box
mkdir -p gpurun_out
export PATH=$PATH:/usr/local/cuda/bin
for mb in 4 5 6; do
  touch paper_1906_11355_b200/csrc/k_interp_mdict.cu
  make -s -C paper_1906_11355_b200/csrc -j8 EXTRA=-DMDICT_BUILD_BATCH=$mb > gpurun_out/mb_build_$mb.log 2>&1 || { echo build $mb failed; tail -5 gpurun_out/mb_build_$mb.log; continue; }
  grep -A2 "k_interp_mdictILi3ELb1ELi16ELb1ELi608" paper_1906_11355_b200/build/k_interp_mdict.ptxas.log | grep -E "registers|spill" | head -2
  for c in 4d l4d; do
    for rep in 1 2; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/mb_${mb}_$c.json 2> gpurun_out/mb_${mb}_$c.err
    python - "$c" "$mb" <<'PY'
import json, sys
c, mb = sys.argv[1:3]
d = json.loads(open(f"gpurun_out/mb_{mb}_{c}.json").read().strip().splitlines()[-1])
p = d.get("passes", {})
print("MB", mb, c, f"{d['value']/1e9:.1f} Gvox/s {d['ms_per_step']:.4f} ms/step", " ".join(f"{k}={v['ms']:.4f}" for k, v in p.items()))
PY
    done
  done
done
