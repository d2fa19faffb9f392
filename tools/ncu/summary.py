import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
keep = ('Duration', 'Elapsed Cycles', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Registers Per Thread',
        'Achieved Occupancy', 'Block Size', 'Grid Size', 'Issue Slots Busy', 'Executed Ipc Active', 'No Eligible', 'Dynamic Shared Memory Per Block',
        'Warp Cycles Per Issued Instruction', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Theoretical Occupancy')
for row in r[1:]:
    name = row[h.index('Metric Name')]
    if name in keep:
        print(f"{row[h.index('Kernel Name')][:30]:30s} {name:40s} {row[h.index('Metric Value')]:>14s} {row[h.index('Metric Unit')]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); h = r[0]; v = r[2]
stalls = []
for i, n in enumerate(h):
    if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued'):
        try: stalls.append((float(v[i].replace(',', '')), n.replace('smsp__pcsamp_warps_issue_stalled_', '')))
        except: pass
stalls.sort(reverse=True)
print('stalls:', ', '.join(f'{n}={int(x)}' for x, n in stalls[:8]))
for i, n in enumerate(h):
    if n in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
        print(n, v[i], r[1][i])
