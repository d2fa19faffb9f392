import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
lines = []
for r in rows[3:]:
    if r and r[0].isdigit():
        try: lines.append((int(r[4]) if r[4] not in ('-', '') else 0, int(r[0]), r[1][:100]))
        except: pass
tot = sum(x[0] for x in lines) or 1
for s, ln, t in sorted(lines, reverse=True)[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}%  L{ln:4d} {t}")
