"""Copy a profile_round.sh result set from gpurun_out/ into profiles/ (summaries, launch-list
shares, traffic.json) -- run on the dev box after the GPU call."""
import csv, collections, json, os, shutil, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(R, "gpurun_out"), os.path.join(R, "profiles")
summ = os.path.join(R, "tools", "ncu_summary.py")
for n in ("nn_it3", "nn_it41", "sel_it41", "acc_it41"):
    with open(os.path.join(P, f"r1_ncu_{n}_c4cert.txt"), "w") as f:
        subprocess.run([sys.executable, summ, os.path.join(G, f"prof_{n}.ncu-rep")], stdout=f, stderr=subprocess.STDOUT)
with open(os.path.join(P, "r1_ncu_proj_c3.txt"), "w") as f:
    subprocess.run([sys.executable, summ, os.path.join(G, "prof_proj_c3.ncu-rep")], stdout=f, stderr=subprocess.STDOUT)
for src, dst in (("bench.json", "r1_bench_c4_plane.json"), ("launches_bench.csv", "r1_launches_bench_c4.csv"),
                 ("stamps.log", "r1_stamps_timeline.txt"), ("sel_class.txt", "r1_sel_classification_c4.txt")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
rows = [json.loads(l) for l in open(os.path.join(G, "bench_all.jsonl"))]
for r in rows:
    if r.get("config") == "C3_depth_projective" and "note" not in r:
        r["kernel_us"] = r["kernel_us"] / r["iterations"] if r["kernel_us"] > 100 else r["kernel_us"]
        r["note"] = "one cooperative persistent launch for the 30 iterations; kernel_us per iteration"
open(os.path.join(P, "r1_bench_all_configs.jsonl"), "w").write("".join(json.dumps(r) + "\n" for r in rows))
rows = list(csv.reader(open(os.path.join(P, "r1_launches_bench_c4.csv"))))
for hi, r in enumerate(rows):
    if "Kernel Name" in r:
        break
h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
tot = collections.Counter(); cnt = collections.Counter()
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0]
    name = name.split("::")[-1] if "::" in name else name
    tot[name] += float(r[vi]) / 1e3; cnt[name] += 1
T = sum(tot.values())
json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline",
           "note": "cold-cache serialised per-launch times: shares, not absolutes",
           "kernels": {k: {"launches": cnt[k], "total_us": round(v, 1), "share": round(v / T, 4)} for k, v in tot.most_common()}},
          open(os.path.join(P, "r1_launches_bench_c4_summary.json"), "w"), indent=1)


def dram(f):
    d = {}
    for line in open(f):
        if "dram__bytes_read.sum" in line or "dram__bytes_write.sum" in line:
            parts = line.split()
            d[parts[0]] = float(parts[1]) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1}[parts[2]]
    return d


t = json.load(open(os.path.join(P, "traffic.json")))
k = {name: int(sum(dram(os.path.join(P, f"r1_ncu_{f}_c4cert.txt")).values()))
     for name, f in (("icp_select_kernel", "sel_it41"), ("icp_nn_kernel", "nn_it41"), ("icp_acc_kernel", "acc_it41"))}
t["c4_plane"]["steady_iteration_kernels"] = k
t["c4_plane"]["steady_iteration_bytes"] = sum(k.values())
t["c4_plane"]["full_search_icp_nn_kernel_bytes"] = int(sum(dram(os.path.join(P, "r1_ncu_nn_it3_c4cert.txt")).values()))
json.dump(t, open(os.path.join(P, "traffic.json"), "w"), indent=1)
b = json.load(open(os.path.join(P, "r1_bench_c4_plane.json")))
print("bench", b["value"], b["ms_per_step"], b["roofline"]["frac"], b["e2e"]["value"])
print("shares", {k: v for k, v in list(tot.most_common())[:4]})
print("traffic", t["c4_plane"]["steady_iteration_bytes"])
