"""Summarise ncu outputs into profiles/: a launch-list share table and per-kernel key metrics.

usage: python scripts/ncu_summary.py <tag> [--launches gpurun_out/launches.csv] [--rep x.ncu-rep ...]
                                     [--workload "<bench config.workload>"]
Writes profiles/<tag>_launches.md, profiles/<tag>_<rep-stem>.md and, with --workload,
profiles/scan_traffic.json[workload] (dram bytes per launch, read by bench.py's roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(path, tag):
    rows = [l for l in open(path) if not l.startswith("==")]
    r = list(csv.reader(io.StringIO("".join(rows))))
    h = r[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.OrderedDict()
    for row in r[1:]:
        if mi is not None and row[mi] != "gpu__time_duration.sum":
            continue   # launch lists may also carry dram byte counters
        name = row[ki]
        v = float(row[vi].replace(",", ""))
        if row[ui] == "usecond":
            v *= 1000.0
        elif row[ui] == "msecond":
            v *= 1e6
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n",
           f"source: `{os.path.relpath(path, ROOT)}`\n",
           "| kernel | launches | total us | avg us | share |", "|---|---:|---:|---:|---:|"]
    for name, (n, ns) in sorted(agg.items(), key=lambda t: -t[1][1]):
        out.append(f"| `{name[:110]}` | {n} | {ns / 1e3:.1f} | {ns / n / 1e3:.2f} | {100 * ns / tot:.1f}% |")
    p = os.path.join(PROF, f"{tag}_launches.md")
    open(p, "w").write("\n".join(out) + "\n")
    print(p)


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Block Size", "Grid Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active",
       "smsp__inst_executed_pipe_tensor", "sm__inst_executed_pipe_tensor"]


def report(rep, tag, workload=None):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    kern = r[1][ki] if len(r) > 1 else "?"
    lines = [f"# {tag}: ncu --set full summary of `{kern[:120]}`\n", f"source: `{os.path.relpath(rep, ROOT)}`\n",
             "| metric | value | unit |", "|---|---:|---|"]
    seen = set()
    for row in r[1:]:
        if row[mi] in WANT and row[mi] not in seen:
            seen.add(row[mi])
            lines.append(f"| {row[mi]} | {row[vi]} | {row[ui]} |")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    vals = {}
    if len(rr) > 2:
        hh, units, v = rr[0], rr[1], rr[2]
        for i, n in enumerate(hh):
            for w in RAW:
                if n.startswith(w):
                    vals[n] = (v[i], units[i])
    lines.append("\nraw counters:\n")
    for n, (v, u) in sorted(vals.items()):
        lines.append(f"- `{n}` = {v} {u}")
    # stall reasons from the source page
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    sr = list(csv.reader(io.StringIO(src)))
    if len(sr) > 2:
        hs = sr[1]
        cols = [i for i, c in enumerate(hs) if c.startswith("stall_") and "Not Issued" not in c]
        tot = collections.Counter()
        for row in sr[2:]:
            for i in cols:
                try:
                    tot[hs[i]] += float(row[i] or 0)
                except ValueError:
                    pass
        s = sum(tot.values()) or 1
        lines.append("\nwarp stall samples (share):\n")
        for n, v in tot.most_common(10):
            lines.append(f"- {n}: {100 * v / s:.1f}%")
    stem = os.path.splitext(os.path.basename(rep))[0]
    p = os.path.join(PROF, f"{tag}_{stem}.md")
    open(p, "w").write("\n".join(lines) + "\n")
    print(p)
    rd = vals.get("dram__bytes_read.sum", (None, None))
    wr = vals.get("dram__bytes_write.sum", (None, None))
    if workload and rd[0] is not None and "scan" in kern:
        def to_bytes(v, u):
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        tb = to_bytes(*rd) + to_bytes(*wr)
        jp = os.path.join(PROF, "scan_traffic.json")
        db = json.load(open(jp)) if os.path.exists(jp) else {}
        db[workload] = {"kernel": kern, "dram_bytes_per_launch": tb, "source": os.path.relpath(p, ROOT)}
        json.dump(db, open(jp, "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--workload", default=None, help="bench workload name: record dram bytes in scan_traffic.json")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    for rep in a.rep:
        report(rep, a.tag, a.workload)
