"""A/B timing of a libcil.so variant (VAR=name: tools/ubench/var_<name>, built by tools/variants.sh;
unset: the in-tree build): C4 50-iteration run (plane and point), C4 stateless iterate at the identity
and the ground truth, C5 iterates, C2 query on the BVH -- device time, L2 flushed, median of 5."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
if os.environ.get("VAR"):
    sys.path.insert(0, os.path.join(root, "tools", "ubench", "var_" + os.environ["VAR"]))
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


out = {}
I4 = d(np.eye(4))
for metric in ("point_to_plane", "point_to_point"):
    w = gen.c4_lidar(metric)
    t = cil.cil_target_build(d(w.target), d(w.target_normals))
    src = d(w.source)
    prm = cil.make_params(metric, w.max_iters, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm)
    out[f"c4_run_{metric[9:]}"] = timed(lambda: cil.cil_icp_run(t, src, I4, prm, ws=ws, want_log=False))
    res_t, _ = cil.cil_icp_run(t, src, I4, prm, ws=ws, want_log=False)
    pose = cil.decode_result(res_t).pose
    if metric == "point_to_plane":
        p1 = cil.make_params(metric, 1, w.max_dist)
        ws1 = cil.alloc_workspace(w.m, p1)
        G4 = d(w.gt_pose)
        out["c4_it_id"] = timed(lambda: cil.cil_icp_iterate(t, src, I4, p1, ws=ws1, want_sys=False))
        out["c4_it_gt"] = timed(lambda: cil.cil_icp_iterate(t, src, G4, p1, ws=ws1, want_sys=False))
        pose_plane = pose
    t.free()
for k in (20, 22):
    w = gen.c5_patches(k)
    t5 = cil.cil_target_build(d(w.target), d(w.target_normals))
    s5 = d(w.source); p5 = cil.make_params("point_to_plane", 1, w.max_dist)
    ws5 = cil.alloc_workspace(w.m, p5)
    out[f"c5_{k}"] = timed(lambda: cil.cil_icp_iterate(t5, s5, I4, p5, ws=ws5, want_sys=False))
    t5.free(); del ws5
w2 = gen.c2_uniform()
t2 = cil.cil_target_build(d(w2.target), None)
q2 = d(w2.source)
out["c2_bvh"] = timed(lambda: cil.cil_nn_query(t2, q2))
print(f"{os.environ.get('VAR', 'tree'):10s} " + " ".join(f"{k} {v:.3f}" for k, v in out.items()) +
      f"  pose[0,3]={pose_plane[0, 3]:.17g}", flush=True)
