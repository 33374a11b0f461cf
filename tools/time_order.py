import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
I4 = d(np.eye(4))
def timed(fn, reps=7):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))
w = gen.c3_depth()
t = cil.cil_target_build(d(w.target), None)
n3, _ = cil.cil_estimate_normals(t, 10, (0.0, 0.0, 0.0)); t.free()
t = cil.cil_target_build(d(w.target), n3)
s = d(w.source); prm = cil.make_params("point_to_plane", 30, w.max_dist); ws = cil.alloc_workspace(w.m, prm)
p1 = cil.make_params("point_to_plane", 1, w.max_dist)
for name, fl in (("auto", 0), ("caller", 16), ("morton", 32)):
    cil.set_debug_flags(fl)
    r = timed(lambda: cil.cil_icp_run(t, s, I4, prm, ws=ws, want_log=False))
    it = timed(lambda: cil.cil_icp_iterate(t, s, I4, p1, ws=ws, want_sys=False))
    res = cil.decode_result(cil.cil_icp_run(t, s, I4, prm, ws=ws, want_log=False)[0])
    print(f"C3 order {name}: run {r:.3f} ms iterate {it:.3f} ms pose03 {res.pose[0,3]:.12f}", flush=True)
w4 = gen.c4_lidar("point_to_plane")
t4 = cil.cil_target_build(d(w4.target), d(w4.target_normals)); s4 = d(w4.source)
prm4 = cil.make_params("point_to_plane", 50, w4.max_dist); ws4 = cil.alloc_workspace(w4.m, prm4)
for name, fl in (("auto", 0), ("caller", 16), ("morton", 32)):
    cil.set_debug_flags(fl)
    r = timed(lambda: cil.cil_icp_run(t4, s4, I4, prm4, ws=ws4, want_log=False), 3)
    print(f"C4 order {name}: run {r:.3f} ms", flush=True)
cil.set_debug_flags(0)
