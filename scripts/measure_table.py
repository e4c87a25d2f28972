"""Markdown table of bench.py JSON lines (one per line in the given files), for DESIGN.md / BASELINE.md.

usage: python scripts/measure_table.py profiles/r02z/sweep.jsonl [more.jsonl ...]"""
import json
import sys


def row(d):
    r = d.get("roofline") or {}
    lp = d.get("latency_pct_ms") or (d.get("latency_ms") if isinstance(d.get("latency_ms"), dict) else {}) or {}
    u = d.get("updates") or {}
    frac = f"{r['frac']:.3f} ({r['bound']})" if r.get("frac") is not None else "—"
    lat = f"{lp.get('p50', 0) * 1e3:.1f} / {lp.get('p95', 0) * 1e3:.1f}" if lp else "—"
    upd = f"; {u['calls_in_timed_region']} update calls × 64 rows ({u['update_call_ms'] * 1e3:.1f} µs each)" if u else ""
    return (f"| {d['config']['workload']}{upd} | {d['ms_per_step'] * 1e3:.1f} µs | {d.get('qps', 0):,.0f} | "
            f"{d['value']:.3g} | {lat} | {frac} | {d['e2e']['value']:.3g} |")


def main():
    print("| workload | step (device) | QPS | items/s | latency p50 / p95 (µs) | roofline frac | e2e items/s |")
    print("|---|---:|---:|---:|---:|---:|---:|")
    for path in sys.argv[1:]:
        for line in open(path):
            line = line.strip()
            if line.startswith("{"):
                d = json.loads(line)
                if "unavailable" in d or d.get("impl") == "reference":
                    continue
                print(row(d))


if __name__ == "__main__":
    main()
