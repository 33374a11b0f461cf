"""Per-CUDA-source-line instruction / stall shares from an ncu report (source page)."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
cur = None; hdr = None
agg = collections.Counter(); stall = collections.Counter(); text = {}
for r in csv.reader(out):
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr is None or not r[0].isdigit(): continue
    ie = r[hdr['Instructions Executed']]
    if ie in ('', '-'): continue
    k = (cur, int(r[0]))
    try:
        agg[k] += int(ie)
    except ValueError:
        continue
    sv = r[hdr["Warp Stall Sampling (All Samples)"]]
    stall[k] += int(sv) if sv.isdigit() else 0
    text[k] = r[1][:90]
tot = sum(agg.values()); ts = max(sum(stall.values()), 1)
print("total warp-instructions", tot)
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{100*v/tot:5.1f}% stall{100*stall[k]/ts:5.1f}% {k[0]}:{k[1]} {text[k]}")
