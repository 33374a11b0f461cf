"""Build and iterate / run times of the small and medium configs (launch-bound index build and
source-order pipelines): C5 2^16..2^20 build + iterate, C1, C3 and C4 build + run.  VAR=name
times tools/ubench/var_<name> (tools/variants.sh).  Device time, L2 flushed, median of 7."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
if os.environ.get("VAR"):
    sys.path.insert(0, os.path.join(root, "tools", "ubench", "var_" + os.environ["VAR"]))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
I4 = d(np.eye(4))


def timed(fn, reps=7):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        if isinstance(r, cil.Target):
            r.free()
    return float(np.median(ts))


out = {}
for k in (16, 18, 20):
    w = gen.c5_patches(k)
    tg, nr, s = d(w.target), d(w.target_normals), d(w.source)
    out[f"c5_{k}_build"] = timed(lambda: cil.cil_target_build(tg, nr))
    t = cil.cil_target_build(tg, nr)
    p1 = cil.make_params("point_to_plane", 1, w.max_dist); ws = cil.alloc_workspace(w.m, p1)
    out[f"c5_{k}_it"] = timed(lambda: cil.cil_icp_iterate(t, s, I4, p1, ws=ws, want_sys=False))
    po = cil.cil_icp_iterate(t, s, I4, p1, ws=ws, want_sys=False)[0]
    out[f"c5_{k}_p03"] = float(po[0, 3])
    t.free()
w = gen.c1_sphere()
tg, nr = d(w.target), d(w.target_normals)
out["c1_build"] = timed(lambda: cil.cil_target_build(tg, nr))
w = gen.c3_depth()
tg = d(w.target)
out["c3_build"] = timed(lambda: cil.cil_target_build(tg, None))
t = cil.cil_target_build(tg, None)
n3, _ = cil.cil_estimate_normals(t, 10, (0.0, 0.0, 0.0)); t.free()
t = cil.cil_target_build(tg, n3)
s = d(w.source); prm = cil.make_params("point_to_plane", 30, w.max_dist); ws = cil.alloc_workspace(w.m, prm)
out["c3_run"] = timed(lambda: cil.cil_icp_run(t, s, I4, prm, ws=ws, want_log=False))
t.free()
w = gen.c4_lidar("point_to_plane")
tg, nr, s = d(w.target), d(w.target_normals), d(w.source)
out["c4_build"] = timed(lambda: cil.cil_target_build(tg, nr))
t = cil.cil_target_build(tg, nr)
prm = cil.make_params("point_to_plane", 50, w.max_dist); ws = cil.alloc_workspace(w.m, prm)
out["c4_run"] = timed(lambda: cil.cil_icp_run(t, s, I4, prm, ws=ws, want_log=False))
res_t, _ = cil.cil_icp_run(t, s, I4, prm, ws=ws, want_log=False)
out["c4_p03"] = float(cil.decode_result(res_t).pose[0, 3])
print(f"{os.environ.get('VAR', 'tree'):10s} " + " ".join(f"{k} {v:.4f}" if "p03" not in k else f"{k} {v:.12g}" for k, v in out.items()), flush=True)
