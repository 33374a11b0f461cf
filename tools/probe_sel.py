"""Per-iteration K_sel classification (diagnostic counters in the workspace state) on C4 or C3
(argv[1]): point-certified, leaf-evaluated, list-evaluated (+ extra list leaves), searched; and
the pose step of every iteration (rotation angle, translation) from the iteration log."""
import os, sys
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
if cfg == "c3":
    w = gen.c3_depth()
    t0 = cil.cil_target_build(d(w.target), None)
    n3, _ = cil.cil_estimate_normals(t0, 10, (0.0, 0.0, 0.0))
    t = cil.cil_target_build(d(w.target), n3)
else:
    w = gen.c4_lidar("point_to_plane")
    t = cil.cil_target_build(d(w.target), d(w.target_normals))
src = d(w.source)
prev = np.zeros(5)
ws = None
poses = []
for k in range(1, w.max_iters + 1):
    prm = cil.make_params("point_to_plane", k, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm) if ws is None else ws
    res, _ = cil.cil_icp_run(t, src, d(np.eye(4)), prm, ws=ws, want_log=False)
    torch.cuda.synchronize()
    P = cil.decode_result(res).pose
    st = ws[176:216].cpu().view(torch.int64).numpy().astype(np.float64)   # searched, pcert, leaf, list, items
    dlt = st - prev
    prev = st
    Pp = poses[-1] if poses else np.eye(4)
    dR = P[:3, :3] @ Pp[:3, :3].T
    ang = np.degrees(np.arccos(np.clip((np.trace(dR) - 1) / 2, -1, 1)))
    poses.append(P)
    m = w.m
    print(f"it {k-1:2d}: searched {dlt[0]/m:6.3f} pointcert {dlt[1]/m:6.3f} leaf {dlt[2]/m:6.3f} list {dlt[3]/m:6.3f} "
          f"extra-list-leaves/pt {dlt[4]/m:6.3f}   step {ang:.5f} deg {np.linalg.norm(P[:3, 3] - Pp[:3, 3]) * 1e3:.4f} mm", flush=True)
