"""Per-source-line stall-reason breakdown (and shared-memory bank conflicts) from an ncu report.

usage: line_stalls.py REPORT [first_line last_line] [top]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[2]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ridx = [h.index(c) for c in reasons]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
conf = h.index("L1 Conflicts Shared N-Way") if "L1 Conflicts Shared N-Way" in h else None
agg = []
for r in rows[3:]:
    if not (r and r[0].isdigit()):
        continue
    ln = int(r[0])
    if not (lo <= ln <= hi):
        continue
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = num(r[si])
    if tot == 0:
        continue
    br = sorted(((num(r[i]), reasons[k][6:]) for k, i in enumerate(ridx)), reverse=True)[:3]
    agg.append((tot, ln, r[1][:60], num(r[ie]), br, r[conf] if conf is not None else ""))
grand = sum(a[0] for a in agg) or 1
for tot, ln, src, n, br, c in sorted(agg, reverse=True)[:top]:
    b = " ".join(f"{name}={int(v)}" for v, name in br if v)
    print(f"{int(tot):6d} {100*tot/grand:5.1f}% L{ln:4d} exec={int(n):9d} conf={c:>5s} | {b} | {src}")
