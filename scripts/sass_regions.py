"""Group an ncu source-page SASS CSV by execution count: how many instructions run how often.
usage: python scripts/sass_regions.py file.src.csv[.gz]"""
import collections, csv, gzip, sys
f = sys.argv[1]
op = gzip.open if f.endswith('.gz') else open
rows = list(csv.reader(op(f, 'rt')))
h = rows[1]
ai, si, ex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
data = rows[2:]
tot = sum(float(r[ex] or 0) for r in data)
by = collections.defaultdict(list)
for r in data:
    by[float(r[ex] or 0)].append(r)
print(f"total executed {tot:.4g}")
for cnt, rs in sorted(by.items(), key=lambda t: -t[0] * len(t[1]))[:25]:
    print(f"count {cnt:12.0f} x {len(rs):4d} instrs = {cnt * len(rs) / tot * 100:5.1f}%  first {rs[0][ai]} {rs[0][si][:50]}")
if len(sys.argv) > 2:
    c = float(sys.argv[2])
    for r in data:
        if float(r[ex] or 0) == c:
            print(r[ai], r[si][:90])
