python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in $CFGS; do
python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/nb_$c.json 2>gpurun_out/nb_$c.err
MCLAHE_NO_NB=1 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/old_$c.json 2>>gpurun_out/nb_$c.err
done
python - <<PY
import json
for c in "$CFGS".split():
    for k in ["nb","old"]:
        try:
            d=json.loads(open(f"gpurun_out/{k}_{c}.json").read().strip().splitlines()[-1])
            print(c,k,round(d["value"]/1e9,2),"K4 GB/s",round(d["roofline"]["achieved"],1), d.get("passes"))
        except Exception as e: print(c,k,"ERR",e)
PY
