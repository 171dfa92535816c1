"""Stall-reason breakdown and shared-memory pipe counters of one kernel in an
ncu report:  python tools/ncu_stalls.py gpurun_out/prof_4d.ncu-rep k_hist_pencil"""
import csv
import subprocess
import sys

rep, kn = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kn}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    f = lambda k: float((d.get(k) or "0").replace(",", "") or 0)
    print(d.get("Kernel Name", "")[:100])
    st = {k: f(k) for k in d if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    print("  stalls:", " ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={x / tot:.0%}"
                              for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:9]))
    keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_bytes.sum"]
    print("  " + " | ".join(f"{k}={d.get(k, '')}" for k in keys if k in d))
