"""C4 iterate at identity / GT pose and the 50-iteration run, overflow handled by the ballot DFS
(flags 0) or by the per-lane DFS (flags 6 = dbg_mode 3); C5 2^22 iterate."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
def tm(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
w = gen.c4_lidar("point_to_plane"); w5 = gen.c5_patches(22)
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src, P0 = d(w.source), d(np.eye(4)); PG = d(w.gt_pose)
prm = cil.make_params("point_to_plane", 50, 1.0); p1 = cil.make_params("point_to_plane", 1, 1.0)
ws = cil.alloc_workspace(w.m, prm)
t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals)); s5 = d(w5.source)
p5 = cil.make_params("point_to_plane", 1, w5.max_dist); ws5 = cil.alloc_workspace(w5.m, p5)
for fl in (0, 6, 0, 6):
    cil.lib().cil_debug_set_flags(fl)
    a = tm(lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, want_log=False))
    b = tm(lambda: cil.cil_icp_iterate(t, src, P0, p1, ws=ws, want_sys=False))
    c = tm(lambda: cil.cil_icp_iterate(t, src, PG, p1, ws=ws, want_sys=False))
    e = tm(lambda: cil.cil_icp_iterate(t5, s5, P0, p5, ws=ws5, want_sys=False))
    print(f"flags {fl}: C4 run {a:.2f} ms, iterate@identity {b:.3f}, @gt {c:.3f}, C5 2^22 {e:.2f}", flush=True)
