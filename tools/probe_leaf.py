"""C4 run / C2 query / C5 iterate times for leaf sizes 4, 8, 16, 32."""
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
w = gen.c4_lidar("point_to_plane"); w2 = gen.c2_uniform(); w5 = gen.c5_patches(22)
for B in (8, 16, 4, 32):
    t = cil.cil_target_build(d(w.target), d(w.target_normals), B)
    src, P0 = d(w.source), d(np.eye(4))
    prm = cil.make_params("point_to_plane", 50, 1.0)
    ws = cil.alloc_workspace(w.m, prm)
    a = tm(lambda: cil.cil_icp_run(t, src, P0, prm, ws=ws, want_log=False))
    p1 = cil.make_params("point_to_plane", 1, 1.0)
    b = tm(lambda: cil.cil_icp_iterate(t, src, P0, p1, ws=ws, want_sys=False))
    t2 = cil.cil_target_build(d(w2.target), None, B); q2 = d(w2.source)
    c = tm(lambda: cil.cil_nn_query(t2, q2))
    t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals), B); s5 = d(w5.source)
    p5 = cil.make_params("point_to_plane", 1, w5.max_dist); ws5 = cil.alloc_workspace(w5.m, p5)
    e = tm(lambda: cil.cil_icp_iterate(t5, s5, P0, p5, ws=ws5, want_sys=False))
    print(f"B={B}: C4 run {a:.2f} ms, C4 iterate@identity {b:.3f} ms, C2 {c:.3f} ms, C5 2^22 {e:.2f} ms", flush=True)
