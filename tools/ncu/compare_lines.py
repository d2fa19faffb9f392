"""Compare two ncu reports of the same kernel line by line (by source TEXT, so
the two builds may number lines differently): warp-stall samples, executed
instructions and shared-memory excessive wavefronts per source line, sorted
by the sample difference.

usage: compare_lines.py A.ncu-rep B.ncu-rep [top]
"""
import csv
import subprocess
import sys
from collections import defaultdict


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[2]
    si = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    ex = h.index("L1 Wavefronts Shared Excessive")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ridx = [h.index(c) for c in reasons]
    agg = defaultdict(lambda: [0.0, 0.0, 0.0, defaultdict(float)])

    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    for r in rows[3:]:
        if not (r and r[0].isdigit()):
            continue
        key = r[1].strip()[:90]
        a = agg[key]
        a[0] += num(r[si])
        a[1] += num(r[ie])
        a[2] += num(r[ex])
        for name, i in zip(reasons, ridx):
            a[3][name] += num(r[i])
    return agg


def main():
    a, b = load(sys.argv[1]), load(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    keys = set(a) | set(b)
    tot_a = sum(v[0] for v in a.values())
    tot_b = sum(v[0] for v in b.values())
    print(f"total stall samples: A {tot_a:.0f}  B {tot_b:.0f}")
    for name in ("stall_long_sb", "stall_short_sb", "stall_wait", "stall_barrier", "stall_no_inst", "stall_mio",
                 "stall_math", "stall_lg", "stall_branch_resolving", "stall_not_selected", "stall_selected",
                 "stall_dispatch", "stall_membar", "stall_sleep", "stall_misc", "stall_drain", "stall_tex"):
        sa = sum(v[3][name] for v in a.values())
        sb = sum(v[3][name] for v in b.values())
        print(f"  {name:24s} A {sa:8.0f}  B {sb:8.0f}  diff {sb - sa:+8.0f}")
    diff = sorted(keys, key=lambda k: -abs((b[k][0] if k in b else 0) - (a[k][0] if k in a else 0)))
    print(f"{'A smp':>8} {'B smp':>8} {'A inst':>10} {'B inst':>10} {'A exc':>8} {'B exc':>8}  source")
    for k in diff[:top]:
        va, vb = a.get(k, [0, 0, 0, {}]), b.get(k, [0, 0, 0, {}])
        print(f"{va[0]:8.0f} {vb[0]:8.0f} {va[1]:10.0f} {vb[1]:10.0f} {va[2]:8.0f} {vb[2]:8.0f}  {k}")


if __name__ == "__main__":
    main()
