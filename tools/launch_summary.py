"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a
bench command: our kernels (namespace mg) by name, launches, mean, share.

    python tools/launch_summary.py gpurun_out/launches_4d.csv > profiles/r01_launches_4d_summary.txt
"""
import csv
import re
import sys
from collections import OrderedDict

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    if not re.search(r"\bmg::|k_(interp|hist|range|mappings|params|thresholds|dict|reset|global|frame)", name):
        continue
    short = re.sub(r"^void ", "", name)
    short = re.sub(r"\(mg::KGeom.*$|\(KGeom.*$|\(const mg::KGeom.*$|\(mg::WS.*$|\(WS.*$", "", short)
    short = short.replace("mg::", "").replace("(int)", "").replace("(bool)", "")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
    rows.append((short, float(r["Metric Value"].replace(",", "")) * scale))
agg = OrderedDict()
for k, us in rows:
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += us
total = sum(a[1] for a in agg.values())
print(f"# {path}: {len(rows)} launches of our kernels, {total / 1e3:.3f} ms total "
      "(cold-cache, serialised per-launch times under ncu: compare SHARES, not absolutes)")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k[:60]:60s} launches={n:4d} mean={us / n:10.3f} us  share={100 * us / total:5.1f}%")
