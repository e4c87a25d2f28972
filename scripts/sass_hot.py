"""Summarise an ncu --page source --print-source sass CSV: hottest instructions by samples/executions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ai, si, smp, ex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot_s = sum(float(r[smp] or 0) for r in data)
tot_e = sum(float(r[ex] or 0) for r in data)
print(f"total samples {tot_s:.0f} executed {tot_e:.0f}")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "samples"
idx = smp if key == "samples" else ex
for r in sorted(data, key=lambda r: -float(r[idx] or 0))[:N]:
    st = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
    print(f"{r[ai]:>6s} {float(r[smp] or 0):7.0f} {float(r[ex] or 0):10.0f}  {r[si][:60]:60s} {st[0][1]}={st[0][0]:.0f} {st[1][1]}={st[1][0]:.0f}")
# stall totals
tot = {}
for r in data:
    for i in stall_cols:
        tot[h[i]] = tot.get(h[i], 0) + float(r[i] or 0)
print(sorted(tot.items(), key=lambda t: -t[1])[:10])
