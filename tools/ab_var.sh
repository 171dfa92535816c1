#!/bin/bash
# A/B of compile-time variants on the GPU box: VARS="name=-DFLAG=1 name2=..." (a
# name with no '=' builds the defaults), AB_SRC = the translation unit to rebuild.
# Per variant: parity subset (AB_TESTS as a -k filter; AB_NO_TESTS=1 skips),
# then device bench lines for AB_CONFIGS.
mkdir -p gpurun_out
export PATH=$PATH:/usr/local/cuda/bin
SRC=${AB_SRC:-k_interp_mdict.cu}
for v in ${VARS:-base}; do
  name=${v%%=*}; flags=""; [ "$v" != "$name" ] && flags=${v#*=}
  for f in $SRC; do touch paper_1906_11355_b200/csrc/$f; done
  make -s -C paper_1906_11355_b200/csrc -j8 EXTRA="$flags" > gpurun_out/var_build_$name.log 2>&1 || { echo "build $name failed"; tail -5 gpurun_out/var_build_$name.log; continue; }
  if [ -z "$AB_NO_TESTS" ]; then
    timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multi_slab.py tests/test_spec_properties.py -m gpu -x -q ${AB_TESTS:+-k "$AB_TESTS"} > gpurun_out/var_tests_$name.log 2>&1
    echo "VAR $name tests rc=$? $(tail -1 gpurun_out/var_tests_$name.log)"
  fi
  for c in ${AB_CONFIGS:-4d}; do
    for rep in 1 2; do
      timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/var_${name}_$c.json 2> gpurun_out/var_${name}_$c.err || { echo "VAR $name $c bench failed"; tail -3 gpurun_out/var_${name}_$c.err; continue; }
      python - "$c" "$name" <<'PY'
import json, sys
c, name = sys.argv[1:3]
d = json.loads(open(f"gpurun_out/var_{name}_{c}.json").read().strip().splitlines()[-1])
p = d.get("passes", {})
print("VAR", name, c, f"{d['value']/1e9:.1f} Gvox/s {d['ms_per_step']:.4f} ms/step", " ".join(f"{k}={v['ms']:.4f}" for k, v in p.items()))
PY
    done
  done
done
