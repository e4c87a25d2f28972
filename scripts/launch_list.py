"""Print the per-launch durations of an ncu --csv --metrics gpu__time_duration.sum log."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if '"Kernel Name"' in l)
r = list(csv.reader(lines[start:]))
h = r[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
for row in r[1:]:
    if len(row) <= vi:
        continue
    v = float(row[vi].replace(",", ""))
    us = v / 1000 if row[ui] == "nsecond" else (v if row[ui] == "usecond" else v * 1000)
    print(f"{us:10.1f} us  {row[ki][:90]}")
