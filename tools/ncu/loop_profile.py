"""Per-loop warp-state samples of one kernel from an ncu report (sass source page).

usage: loop_profile.py REPORT OBJ FUNC_SUBSTR [min_len]
Loops are found statically in the object's SASS (backward branches, as
tools/sass_loops.py); ncu addresses are matched by offset from the function
start. For each loop prints body length, executions of the loop head, samples
and the top stall reasons (samples inside nested loops count in the outer).
"""
import csv
import re
import subprocess
import sys
from collections import Counter

rep, obj, fn = sys.argv[1], sys.argv[2], sys.argv[3]
min_len = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ai = h.index("Address")
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") or c.startswith("smsp__pcsamp")]
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ai], 16), r))
    except (ValueError, IndexError):
        pass
base = recs[0][0]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
body = next(f for f in re.split(r"\n\s+Function : ", sass) if fn in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
by_off = {a - base: r for a, r in recs}
tot = sum(int(r[si]) for _, r in recs) or 1
print(f"total samples {tot}; stall columns: {[c for _, c in stall_cols][:3]}...")
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA (?:`\(.*?\))?\s*0x([0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt < a and tgt in addr_idx and i - addr_idx[tgt] + 1 >= min_len:
        n = i - addr_idx[tgt] + 1
        samples = 0
        reasons = Counter()
        head = by_off.get(tgt)
        for off in range(tgt, a + 16, 16):
            r = by_off.get(off)
            if r is None:
                continue
            samples += int(r[si] or 0)
            for ci, c in stall_cols:
                try:
                    reasons[c.replace("stall_", "")] += int(r[ci] or 0)
                except ValueError:
                    pass
        ex = head[ie] if head else "?"
        top = ", ".join(f"{k}={v}" for k, v in reasons.most_common(6) if v)
        print(f"0x{tgt:x}..0x{a:x} n={n:5d} head_exec={ex:>8s} samples={samples:6d} ({100*samples/tot:4.1f}%) | {top}")
