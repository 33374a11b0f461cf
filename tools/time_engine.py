"""Engine timings of the libcil.so first on sys.path (variants): C4 stateless iterate at the
identity and the ground truth, C2 BVH query, C5 2^22 iterate (L2 flushed, median of 5)."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.append(root)
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.path.dirname(os.path.dirname(cil.__file__)).split("/")[-1]


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = {}
w = gen.c4_lidar("point_to_plane")
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src = d(w.source)
prm = cil.make_params("point_to_plane", 1, w.max_dist)
ws = cil.alloc_workspace(w.m, prm)
for name, P in (("c4_it_id", np.eye(4)), ("c4_it_gt", w.gt_pose)):
    Pd = d(P)
    out[name] = timed(lambda: cil.cil_icp_iterate(t, src, Pd, prm, ws=ws, want_sys=False))
del t, src, ws
w2 = gen.c2_uniform()
t2 = cil.cil_target_build(d(w2.target), None)
q2 = d(w2.source)
out["c2_bvh"] = timed(lambda: cil.cil_nn_query(t2, q2))
del t2, q2
w5 = gen.c5_patches(22)
t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals))
s5 = d(w5.source)
prm5 = cil.make_params("point_to_plane", 1, w5.max_dist)
ws5 = cil.alloc_workspace(w5.m, prm5)
P0 = d(np.eye(4))
out["c5_22_it"] = timed(lambda: cil.cil_icp_iterate(t5, s5, P0, prm5, ws=ws5, want_sys=False))
print(tag, " ".join(f"{k} {v:.3f} ms" for k, v in out.items()), flush=True)
