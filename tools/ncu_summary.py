"""Summarise an ncu report: per-opcode stall/executed shares, hottest SASS
lines, key speed-of-light metrics, DRAM traffic.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep k_interp
"""
import csv, sys, subprocess
from collections import Counter
rep, kn = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kn}", "--print-source", "sass"], capture_output=True, text=True).stdout
allrows = list(csv.reader(out.splitlines()))
# several kernels may match: keep the section with the most stall samples
secs, cur = [], None
for r in allrows:
    if r and r[0] == "Kernel Name":
        cur = []
        secs.append(cur)
    if cur is not None:
        cur.append(r)
def _samples(sec):
    try:
        i = sec[1].index("Warp Stall Sampling (All Samples)")
        return sum(int(x[i] or 0) for x in sec[2:] if len(x) > i and x[i].isdigit())
    except Exception:
        return 0
rows = max(secs, key=_samples)
print(rows[0][1][:110])
hdr = rows[1]
si, st, ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try: data.append((int(r[st] or 0), int(r[ex] or 0), r[si]))
    except: pass
tot = sum(d[0] for d in data) or 1; totex = sum(d[1] for d in data) or 1
print(kn, "samples", tot, "executed", totex)
c = Counter(); e = Counter()
for s, x, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith('@'): op = src.split()[1]
    op = op.split('.')[0]; c[op] += s; e[op] += x
print(" ".join(f"{op}:{100*s/tot:.0f}%/{100*e[op]/totex:.0f}%" for op, s in c.most_common(18)))
for s, x, src in sorted(data, reverse=True)[:12]: print("  ", s, x, src[:90])
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "--kernel-name", f"regex:{kn}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]; mi, vi = h.index("Metric Name"), h.index("Metric Value")
want = {'Duration','DRAM Throughput','Compute (SM) Throughput','Issued Ipc Active','Achieved Occupancy','Registers Per Thread','L1/TEX Hit Rate','L2 Hit Rate','Mem Busy','Max Bandwidth','Local Memory Spilling Requests'}
print(" | ".join(f"{r[mi]}={r[vi]}" for r in rows[1:] if r[mi] in want))
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", f"regex:{kn}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    vals = {name: r[i] for i, name in enumerate(h)}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
            "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
    print("raw: " + " | ".join(f"{k}={vals.get(k)}" for k in keys))
