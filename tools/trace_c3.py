"""Engine trace statistics on C3 (depth frame, GPU PCA normals): stateless iterate at the
identity and the ground truth, a warm uncertified run, and the certified run's timeline."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
from scipy.spatial.transform import Rotation

w = gen.c3_depth()
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t0 = cil.cil_target_build(d(w.target), None)
nrm, _ = cil.cil_estimate_normals(t0, 10, (0.0, 0.0, 0.0))
t = cil.cil_target_build(d(w.target), nrm)
src = d(w.source)
f32 = lambda a: np.asarray(a, np.int32).view(np.float32)


def pose_frac(f):
    rv = Rotation.from_matrix(w.gt_pose[:3, :3]).as_rotvec() * f
    T = np.eye(4); T[:3, :3] = Rotation.from_rotvec(rv).as_matrix(); T[:3, 3] = w.gt_pose[:3, 3] * f
    return T


def summarize(tag, tr):
    fl = tr[:, 0]
    nF, items = tr[:, 4], tr[:, 6]
    lane0 = np.arange(len(tr)) % 32 == 0
    q = lambda x: np.percentile(x, [50, 90, 99]).round(1).tolist()
    print(tag, "normal", round((fl & 1).mean(), 4), "outlier", round(((fl >> 1) & 1).mean(), 4),
          "overflow", round(((fl >> 2) & 1).mean(), 4), "sparse", round(((fl >> 3) & 1).mean(), 4),
          "| nF mean", round(nF[lane0].mean(), 1), "p50/90/99", q(nF[lane0]),
          "| items/query mean", round(items.mean(), 2), "p50/90/99", q(items),
          "| r p50/90/99", q(f32(tr[:, 1])), "| keyrange/32 p50/90", q((tr[lane0, 3] - tr[lane0, 2]) / 8.0)[:2],
          "| best d p50/90", q(np.sqrt(np.maximum(f32(tr[:, 7]), 0)))[:2], flush=True)
    ck = tr[lane0, 8:13].astype(np.float64)
    tot = ck.sum(0)
    print("    clock share A B C DE F:", (tot / tot.sum()).round(3).tolist(), "mean clocks/packet",
          round(tot.sum() / lane0.sum()), flush=True)


prm = cil.make_params("point_to_plane", 1, w.max_dist)
tr = torch.zeros(w.m * 16, dtype=torch.int32, device="cuda")
for f in (0.0, 1.0):
    cil.lib().cil_debug_engine_trace(tr.data_ptr())
    cil.cil_icp_iterate(t, src, d(pose_frac(f)), prm, want_sys=False)
    torch.cuda.synchronize()
    cil.lib().cil_debug_engine_trace(None)
    summarize(f"iterate pose {f}", tr.cpu().numpy().reshape(-1, 16))
for order in (0, 16):
    cil.lib().cil_debug_set_flags(order)
    for k in (5, 20):
        pk = cil.make_params("point_to_plane", k, w.max_dist)
        ws = cil.alloc_workspace(w.m, pk)
        tr[:] = 0
        cil.lib().cil_debug_engine_trace(tr.data_ptr())
        cil.cil_icp_run(t, src, d(np.eye(4)), pk, ws=ws)
        torch.cuda.synchronize()
        cil.lib().cil_debug_engine_trace(None)
        a = tr.cpu().numpy().reshape(-1, 16)
        sel = a[:, 13] == k - 1
        summarize(f"cert run (flags {order}) iteration {k - 1} [{sel.sum()} slots]", a[sel] if sel.any() else a)
cil.lib().cil_debug_set_flags(0)
