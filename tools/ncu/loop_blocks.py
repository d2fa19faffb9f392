"""List the hot SASS loops of a kernel in an ncu report: contiguous address
runs with one execution count, with instruction count, stall samples and the
mix of opcodes (design evidence for per-step instruction budgets).

usage: loop_blocks.py REPORT [min_exec]
"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ai, si, wi, ie = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index(
    "Instructions Executed")
ins = []
for r in rows[hdr + 1:]:
    try:
        ins.append((int(r[ai], 16), r[si], int(r[wi] or 0), int(r[ie] or 0)))
    except (ValueError, IndexError):
        pass
runs = []
cur = None
for a, src, st, ex in ins:
    if cur and ex == cur["exec"]:
        cur["n"] += 1
        cur["stall"] += st
        cur["ops"][src.split()[0] if not src.startswith("@") else src.split()[1]] += 1
    else:
        if cur:
            runs.append(cur)
        cur = {"start": a, "exec": ex, "n": 1, "stall": st, "ops": Counter()}
        cur["ops"][src.split()[0] if src and not src.startswith("@") else (src.split()[1] if src else "?")] += 1
runs.append(cur)
for r in runs:
    if r["exec"] >= min_exec and r["n"] >= 8:
        top = ", ".join(f"{k}:{v}" for k, v in r["ops"].most_common(10))
        print(f"{r['start']:#x} exec={r['exec']:8d} n={r['n']:4d} stall={r['stall']:6d} | {top}")
