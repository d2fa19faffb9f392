"""Static SASS loop finder: prints every backward branch (loop) of one
function with its body length and opcode mix (no GPU needed).

usage: sass_loops.py OBJ FUNCTION_SUBSTRING [min_len]
"""
import re
import subprocess
import sys
from collections import Counter

obj, fn = sys.argv[1], sys.argv[2]
min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if fn in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA (?:`\(.*?\))?\s*0x([0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt < a and tgt in addr_idx:
        j = addr_idx[tgt]
        n = i - j + 1
        if n >= min_len:
            ops = Counter(t.split()[0] if not t.startswith("@") else t.split()[1] for _, t in ins[j:i + 1])
            top = ", ".join(f"{k}:{v}" for k, v in ops.most_common(12))
            print(f"loop {tgt:#x}..{a:#x} n={n}: {top}")
