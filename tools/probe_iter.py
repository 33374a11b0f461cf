"""Timing probe for the ICP iteration on C4 (GPU box): stateless iterate at the identity and
at the ground-truth pose, cil_icp_run with and without the certified warm start (per-kernel
event times and the number of full searches), and the C2 exact-NN query."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

metric = sys.argv[1] if len(sys.argv) > 1 else "point_to_plane"
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = gen.c4_lidar(metric)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
tgt, nrm, src = d(w.target), d(w.target_normals), d(w.source)
t = cil.cil_target_build(tgt, nrm, leaf)
prm = cil.make_params(metric, 50, 1.0)
ws = cil.alloc_workspace(w.m, prm)
ev = lambda: torch.cuda.Event(enable_timing=True)


def pose_frac(f):
    from scipy.spatial.transform import Rotation
    rv = Rotation.from_matrix(w.gt_pose[:3, :3]).as_rotvec() * f
    T = np.eye(4); T[:3, :3] = Rotation.from_rotvec(rv).as_matrix(); T[:3, 3] = w.gt_pose[:3, 3] * f
    return T


for f in (0.0, 1.0):
    P = d(pose_frac(f))
    for _ in range(2): cil.cil_icp_iterate(t, src, P, prm, ws=ws, want_sys=False)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(5): cil.cil_icp_iterate(t, src, P, prm, ws=ws, want_sys=False)
    e1.record(); torch.cuda.synchronize()
    print(f"iterate pose {f}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)

P0 = d(np.eye(4))
for cert, gap in ((True, (0.001, 0.005, 16.0)), (False, 0.0)):
    cil.set_certificates(cert)
    if cert: cil.set_cert_skin(*gap)
    for k in (1, 2, 5, 10, 20, 30, 50):
        pk = cil.make_params(metric, k, 1.0)
        cil.cil_icp_run(t, src, P0, pk, ws=ws, want_log=False)
        torch.cuda.synchronize()
        cil.profile_enable(True); cil.profile_read()
        e0, e1 = ev(), ev()
        e0.record(); res, _ = cil.cil_icp_run(t, src, P0, pk, ws=ws, want_log=False); e1.record(); torch.cuda.synchronize()
        pr = cil.profile_read(); cil.profile_enable(False)
        r = cil.decode_result(res)
        print(f"run cert={int(cert)} gap {gap} iters {k}: {e0.elapsed_time(e1):.3f} ms  sel {pr['sel_ms']:.3f} nn {pr['nn_ms']:.3f} "
              f"acc {pr['acc_ms']:.3f}  searched {cil.run_searched(ws)} ({cil.run_searched(ws)/w.m:.2f} full-equiv)  "
              f"rmse {r.rmse:.6f} n_corr {r.n_corr}", flush=True)
cil.set_certificates(True)
w2 = gen.c2_uniform()
t2 = cil.cil_target_build(d(w2.target), None, leaf)
q2 = d(w2.source)
for _ in range(2): cil.cil_nn_query(t2, q2)
torch.cuda.synchronize()
e0, e1 = ev(), ev()
e0.record()
for _ in range(5): cil.cil_nn_query(t2, q2)
e1.record(); torch.cuda.synchronize()
print("c2 nn ms", e0.elapsed_time(e1) / 5)
