"""SASS opcode histogram of the library's hot kernels (cuobjdump -sass on the built liblinr.so).

usage: python scripts/sass_hist.py [out.md]
Evidence that the batched path runs on tcgen05 (UTCHMMA / UTCIMMA, LDTM, UTMALDG) and that the
GEMV path uses LDGSTS + LDSM + HMMA/IMMA; the kernel list is the hot path's."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2407_13218_b200", "liblinr.so")
WANT = [  # (label, regex on the mangled name)
    ("scan_ws_kernel<bf16,128,1> (GEMV ring scan, c2)", r"scan_ws_kernelILi2ELi128ELi1E"),
    ("scan_ws_kernel<i8,64,1> (GEMV ring scan, c4 shard)", r"scan_ws_kernelILi3ELi64ELi1E"),
    ("tc_scan_kernel<bf16,128,256> (tcgen05 batched, c2 B=256)", r"tc_scan_kernelILi2ELi128ELi256E"),
    ("tc_scan_kernel<i8,64,256> (tcgen05 kind::i8)", r"tc_scan_kernelILi3ELi64ELi256E"),
    ("merge_kernel", r"merge_kernel"),
    ("code_hist_kernel (quantised pass 1)", r"code_hist_kernel"),
]
KEY = ["UTCHMMA", "UTCIMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "SYNCS", "LDGSTS", "LDSM", "HMMA", "IMMA",
       "LDG", "LDS", "STS", "STG", "SHFL", "VOTE", "REDUX", "ATOMS", "ATOMG", "BAR", "FMNMX", "SHF", "BRA"]


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "sass_histogram.md")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            funcs[cur][m.group(1)] += 1
    lines = ["# SASS opcode histogram of the hot kernels (static instruction counts)", "",
             f"source: `cuobjdump -sass paper_2407_13218_b200/liblinr.so` ({os.path.basename(__file__)}); "
             "counts are static (instructions in the binary), not executions.", ""]
    lines.append("| kernel | total | " + " | ".join(KEY) + " |")
    lines.append("|---|---:|" + "---:|" * len(KEY))
    for label, rx in WANT:
        names = [f for f in funcs if re.search(rx, f)]
        if not names:
            continue
        c = collections.Counter()
        for f in names:
            c.update(funcs[f])
        tot = sum(c.values())
        lines.append(f"| {label} ({len(names)} fn) | {tot} | " + " | ".join(str(c.get(k, 0)) for k in KEY) + " |")
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
