"""(Modes 1-2 need a trace build: tools/variants.sh trace "-DCIL_TRACE=1", then PYTHONPATH=tools/ubench/var_trace.)
Engine timings under the diagnostic engine modes (cil_debug_set_flags bits 1-2): 0 = packet
phases, 1 = every lane through the ballot DFS, 2 = no outlier cap.  C4 iterate at the identity and
the ground truth, C2 BVH query, C5 2^20 / 2^22 iterate (L2 flushed, median of 5)."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


cases = []
w = gen.c4_lidar("point_to_plane")
t4 = cil.cil_target_build(d(w.target), d(w.target_normals)); s4 = d(w.source)
p4 = cil.make_params("point_to_plane", 1, w.max_dist); ws4 = cil.alloc_workspace(w.m, p4)
for name, P in (("c4_it_id", np.eye(4)), ("c4_it_gt", w.gt_pose)):
    Pd = d(P)
    cases.append((name, lambda Pd=Pd: cil.cil_icp_iterate(t4, s4, Pd, p4, ws=ws4, want_sys=False)))
w2 = gen.c2_uniform()
t2 = cil.cil_target_build(d(w2.target), None); q2 = d(w2.source)
cases.append(("c2_bvh", lambda: cil.cil_nn_query(t2, q2)))
for logn in (20, 22):
    w5 = gen.c5_patches(logn)
    t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals)); s5 = d(w5.source)
    p5 = cil.make_params("point_to_plane", 1, w5.max_dist); ws5 = cil.alloc_workspace(w5.m, p5)
    P0 = d(np.eye(4))
    cases.append((f"c5_{logn}_it", lambda t5=t5, s5=s5, p5=p5, ws5=ws5, P0=P0: cil.cil_icp_iterate(t5, s5, P0, p5, ws=ws5, want_sys=False)))
for mode in (0, 1, 2):
    cil.lib().cil_debug_set_flags(mode << 1)
    print(f"mode {mode}: " + " ".join(f"{n} {timed(f):.3f}" for n, f in cases), flush=True)
cil.lib().cil_debug_set_flags(0)
