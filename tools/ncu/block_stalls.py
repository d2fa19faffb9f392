"""Per-instruction stall breakdown of one SASS block (address range) of an ncu report.

usage: block_stalls.py REPORT START_ADDR_HEX N
"""
import csv
import subprocess
import sys
from collections import Counter

rep, start, n = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ai, si = h.index("Address"), h.index("Source")
scols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
ins = [r for r in rows[hdr + 1:] if len(r) > si]
idx = next(i for i, r in enumerate(ins) if int(r[ai], 16) == start)
tot = Counter()
for r in ins[idx: idx + n]:
    parts = []
    for i, c in scols:
        try:
            v = int(float(r[i] or 0))
        except ValueError:
            v = 0
        if v:
            tot[c] += v
            parts.append(f"{c[6:]}={v}")
    print(f"{r[ai][-5:]} {r[si][:60]:60s} {' '.join(parts)}")
print("TOTAL", ", ".join(f"{k[6:]}={v}" for k, v in tot.most_common()))
