"""A/B of the leaf neighbour lists: C4 50-iteration run, C4 stateless iterate at the
identity / ground truth, C5 iterates, C2 BVH query and the index build, with lists of K entries
(K = 0: none built) -- device time, L2 flushed, median of 5."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
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


Ks = [int(k) for k in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["-1", "32", "64", "128"])]
w = gen.c4_lidar("point_to_plane")
tg, tn, src = d(w.target), d(w.target_normals), d(w.source)
prm1 = cil.make_params("point_to_plane", 1, w.max_dist)
prm = cil.make_params("point_to_plane", w.max_iters, w.max_dist)
ws1 = cil.alloc_workspace(w.m, prm1)
ws = cil.alloc_workspace(w.m, prm)
I4, G4 = d(np.eye(4)), d(w.gt_pose)
w5 = {k: gen.c5_patches(k) for k in (20, 22)}
w2 = gen.c2_uniform()
for K in Ks:
    out = {}
    out["build"] = timed(lambda: cil.cil_target_build(tg, tn, leaf_lists=K))
    t = cil.cil_target_build(tg, tn, leaf_lists=K)
    out["c4_run"] = timed(lambda: cil.cil_icp_run(t, src, I4, prm, ws=ws, want_log=False))
    res_t, _ = cil.cil_icp_run(t, src, I4, prm, ws=ws, want_log=False)
    r = cil.decode_result(res_t)
    out["c4_it_id"] = timed(lambda: cil.cil_icp_iterate(t, src, I4, prm1, ws=ws1, want_sys=False))
    out["c4_it_gt"] = timed(lambda: cil.cil_icp_iterate(t, src, G4, prm1, ws=ws1, want_sys=False))
    t.free()
    for k, w_ in w5.items():
        t5 = cil.cil_target_build(d(w_.target), d(w_.target_normals), leaf_lists=K)
        s5 = d(w_.source); p5 = cil.make_params("point_to_plane", 1, w_.max_dist)
        ws5 = cil.alloc_workspace(w_.m, p5)
        out[f"c5_{k}"] = timed(lambda: cil.cil_icp_iterate(t5, s5, I4, p5, ws=ws5, want_sys=False))
        t5.free(); del ws5
    t2 = cil.cil_target_build(d(w2.target), None, leaf_lists=K)
    q2 = d(w2.source)
    out["c2_bvh"] = timed(lambda: cil.cil_nn_query(t2, q2))
    t2.free()
    print(f"K={K:4d} " + " ".join(f"{k} {v:.3f}" for k, v in out.items()) + f"  pose[0,3]={r.pose[0,3]:.17g}", flush=True)
