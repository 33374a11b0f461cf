"""Timing/diagnostic probe for the ICP iteration on C4 (GPU box)."""
import ctypes as C
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
from scipy.spatial.transform import Rotation

L = cil.lib()
L.cil_debug_nn_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_float, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
metric = sys.argv[1] if len(sys.argv) > 1 else "point_to_plane"
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = gen.c4_lidar(metric)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
tgt, nrm, src = d(w.target), d(w.target_normals), d(w.source)
t = cil.cil_target_build(tgt, nrm, leaf)
prm = cil.make_params(metric, 50, 1.0)
ws = cil.alloc_workspace(w.m, prm)
NNPOS_OFF = 256 + ((1184 * 32 * 8 + 255) // 256) * 256
ev = lambda: torch.cuda.Event(enable_timing=True)

def pose_frac(f):
    rv = Rotation.from_matrix(w.gt_pose[:3, :3]).as_rotvec() * f
    T = np.eye(4); T[:3, :3] = Rotation.from_rotvec(rv).as_matrix(); T[:3, 3] = w.gt_pose[:3, 3] * f
    return T

def stats(P, hint):
    n_ = torch.empty(w.m, dtype=torch.int32, device="cuda"); l_ = torch.empty_like(n_); v_ = torch.empty_like(n_)
    rc = L.cil_debug_nn_stats(t.handle, src.data_ptr(), w.m, P.data_ptr(), C.c_float(1.0),
                              None if hint is None else hint.data_ptr(), n_.data_ptr(), l_.data_ptr(), v_.data_ptr(), None)
    torch.cuda.synchronize()
    a = [x.cpu().numpy() for x in (n_, l_, v_)]
    return {k: (round(float(x.mean()), 1), int(np.median(x)), int(np.quantile(x, .99))) for k, x in zip(("nodes", "leaves", "levels"), a)} | {"rc": rc}

for f in (0.0, 1.0):
    P = d(pose_frac(f))
    for _ in range(2): cil.cil_icp_iterate(t, src, P, prm, ws=ws, want_sys=False)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(5): cil.cil_icp_iterate(t, src, P, prm, ws=ws, want_sys=False)
    e1.record(); torch.cuda.synchronize()
    hint = ws[NNPOS_OFF:NNPOS_OFF + 4 * w.m].view(torch.int32).clone()
    print(f"pose {f}: iterate ms {e0.elapsed_time(e1)/5:.3f} cold {stats(P, None)} warm {stats(P, hint)}", flush=True)

P0 = d(np.eye(4))
for k in (1, 2, 5, 10, 20, 50):
    pk = cil.make_params(metric, k, 1.0)
    cil.cil_icp_run(t, src, P0, pk, ws=ws, want_log=False)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(); cil.cil_icp_run(t, src, P0, pk, ws=ws, want_log=False); e1.record(); torch.cuda.synchronize()
    print("run", k, "iters ms", round(e0.elapsed_time(e1), 3), flush=True)
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
