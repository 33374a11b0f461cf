"""Summarise an ncu report (details + SASS hot spots) for profiles/."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(det.splitlines())); h = r[0]; I = {k: i for i, k in enumerate(h)}
want = ['Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Avg. Active Threads Per Warp', 'Achieved Active Warps Per SM',
        'Theoretical Occupancy', 'Executed Instructions', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'DRAM Throughput', 'Registers Per Thread',
        'Warp Cycles Per Issued Instruction', 'Branch Efficiency', 'Mem Busy', 'Max Bandwidth', 'Memory Throughput', 'Grid Size', 'Block Size']
print("kernel:", r[1][I['Kernel Name']][:100])
for row in r[1:]:
    if any(row[I['Metric Name']] == w for w in want):
        print("  ", row[I['Metric Name']].ljust(40), row[I['Metric Value']], row[I['Metric Unit']])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rr = list(csv.reader(raw)); hh = rr[0]
vals = rr[2] if len(rr) > 2 else rr[1]
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__inst_executed_pipe_fma.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"):
    if k in hh:
        print("  ", k.ljust(40), vals[hh.index(k)], rr[1][hh.index(k)])
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(sass)); h = rows[1]; I = {k: i for i, k in enumerate(h)}; data = rows[2:]
tot_s = sum(int(x[I['Warp Stall Sampling (All Samples)']] or 0) for x in data)
tot_i = sum(int(x[I['Instructions Executed']] or 0) for x in data)
byop, byops = collections.Counter(), collections.Counter()
for x in data:
    toks = x[I['Source']].split()
    if not toks: continue
    op = (toks[1] if toks[0].startswith('@') else toks[0]).split('.')[0]
    byop[op] += int(x[I['Instructions Executed']] or 0); byops[op] += int(x[I['Warp Stall Sampling (All Samples)']] or 0)
print("  warp-instructions executed", tot_i, " stall samples", tot_s)
for op, c in byop.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    print("   ", op.ljust(10), str(c).rjust(12), f"{100*c/tot_i:5.1f}%  stall {100*byops[op]/tot_s:5.1f}%")
