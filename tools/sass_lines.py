"""Attribute ncu per-instruction counters of one kernel to CUDA source lines.
usage: python tools/sass_lines.py <report.ncu-rep> <mangled-kernel-substring> <cubin>"""
import collections, csv, re, subprocess, sys

rep, kname, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
# find the function section, collect offset -> (file, line)
cur_fn, cur_loc, off2loc = None, None, {}
for ln in dis:
    m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"\s*(_Z\S+):\s*$", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_loc = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and kname in cur_fn:
        off2loc[int(m.group(1), 16)] = cur_loc
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                      capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(sass)); h = rows[1]; I = {k: i for i, k in enumerate(h)}; data = rows[2:]
base = min(int(r[I["Address"]], 16) for r in data)
agg, aggs = collections.Counter(), collections.Counter()
for r in data:
    off = int(r[I["Address"]], 16) - base
    loc = off2loc.get(off, ("?", 0))
    agg[loc] += int(r[I["Instructions Executed"]] or 0)
    aggs[loc] += int(r[I["Warp Stall Sampling (All Samples)"]] or 0)
tot, tots = sum(agg.values()), sum(aggs.values())
print("mapped offsets:", len(off2loc), "instructions:", tot)
src = {}
for (f, l), c in agg.most_common(45):
    print(f"{100*c/tot:5.1f}% inst {100*aggs[(f,l)]/max(tots,1):5.1f}% stall  {f}:{l}")
