"""Per-SASS-line stall reasons of one kernel (ncu source page):
    python tools/ncu_lines.py REP KERNEL_REGEX [REASON] [N]
Prints the N lines with the most samples of REASON (default: all samples)
and the reason totals."""
import csv
import subprocess
import sys

rep, kn = sys.argv[1], sys.argv[2]
reason = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kn}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Address":
        cur = [r]
        secs.append(cur)
    elif cur is not None and r:
        cur.append(r)
sec = max(secs, key=len)
h = sec[0]
ix = {c: i for i, c in enumerate(h)}
def num(r, c):
    try:
        return float(r[ix[c]] or 0)
    except Exception:
        return 0.0
data = sec[1:]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: sum(num(r, c) for r in data) for c in reasons}
T = sum(tot.values()) or 1
print(" ".join(f"{c[6:]}={v / T:.0%}" for c, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v / T > 0.005))
key = reason if reason in ix else "stall_" + reason
for i, r in sorted(enumerate(data), key=lambda t: -num(t[1], key))[:N]:
    top = sorted(((num(r, c), c[6:]) for c in reasons), reverse=True)[:3]
    print(f"{i:5d} {r[ix['Address']]:>6} {num(r, key):6.0f} ex={num(r, 'Instructions Executed'):9.0f} "
          f"{r[ix['Source']][:60]:60s} " + " ".join(f"{c}:{v:.0f}" for v, c in top if v))
