"""Top SASS instructions by stall samples from an ncu report (source page, sass view)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ai, si = h.index("Address"), h.index("Source")
wi = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed") if "Instructions Executed" in h else None
items = []
for r in rows[hdr + 1:]:
    try:
        items.append((int(r[wi]), r[ai], r[si], r[ie] if ie is not None else ""))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in items) or 1
for s, a, src, n in sorted(items, reverse=True)[:top]:
    print(f"{s:6d} {100 * s / tot:5.1f}% {a} {src[:70]:70s} exec={n}")
