"""Print SASS instructions (address order) around an anchor mnemonic with stall samples."""
import csv
import subprocess
import sys

rep, anchor = sys.argv[1], sys.argv[2]
before = int(sys.argv[3]) if len(sys.argv) > 3 else 20
after = int(sys.argv[4]) if len(sys.argv) > 4 else 200
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
ins = [r for r in rows[hdr + 1:] if len(r) > wi]
idx = next(i for i, r in enumerate(ins) if anchor in r[si])
for r in ins[max(0, idx - before): idx + after]:
    print(f"{r[ai][-5:]} {r[wi]:>6s} {r[ie]:>8s}  {r[si][:80]}")
