"""(Needs a trace build: tools/variants.sh trace "-DCIL_TRACE=1", then PYTHONPATH=tools/ubench/var_trace.)
Engine trace statistics on C4 (GPU box): per-query packet phases at the identity and the
ground-truth pose (stateless iterate, cold hints) and in a warm run (iteration k)."""
import sys, os
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))   # (a variant on PYTHONPATH wins)
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
from scipy.spatial.transform import Rotation

metric = "point_to_plane"
w = gen.c4_lidar(metric)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals))
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
          "overflow", round(((fl >> 2) & 1).mean(), 4),
          "| per packet nF mean", round(nF[lane0].mean(), 1), "p50/90/99", q(nF[lane0]),
          "| items/query mean", round(items.mean(), 2), "p50/90/99", q(items),
          "| r p50/90/99", q(f32(tr[:, 1])), "| keyrange/32 p50/90", q((tr[lane0, 3] - tr[lane0, 2]) / 8.0)[:2], flush=True)
    ck = tr[lane0, 8:13].astype(np.float64)
    tot = ck.sum(0)
    print("    clock share A(hint) B(box) C(range+walk) DE(tests+items) F(dfs):", (tot / tot.sum()).round(3).tolist(),
          "mean clocks/packet", round(tot.sum() / lane0.sum()), flush=True)

prm = cil.make_params(metric, 1, 1.0)
tr = torch.zeros(w.m * 16, dtype=torch.int32, device="cuda")
for f in (0.0, 1.0):
    cil.lib().cil_debug_engine_trace(tr.data_ptr())
    cil.cil_icp_iterate(t, src, d(pose_frac(f)), prm, want_sys=False)
    torch.cuda.synchronize()
    cil.lib().cil_debug_engine_trace(None)
    summarize(f"iterate pose {f}", tr.cpu().numpy().reshape(-1, 16))
cil.set_certificates(False)
for k in (2, 10, 30):
    pk = cil.make_params(metric, k - 1, 1.0)
    ws = cil.alloc_workspace(w.m, pk)
    cil.cil_icp_run(t, src, d(np.eye(4)), pk, ws=ws)
    torch.cuda.synchronize()
    # one more warm iteration, traced: a run of k iterations traces every iteration; keep the last
    pk = cil.make_params(metric, k, 1.0)
    cil.lib().cil_debug_engine_trace(tr.data_ptr())
    cil.cil_icp_run(t, src, d(np.eye(4)), pk, ws=ws)
    torch.cuda.synchronize()
    cil.lib().cil_debug_engine_trace(None)
    summarize(f"run (no cert) iteration {k}", tr.cpu().numpy().reshape(-1, 16))

cil.set_certificates(True)
for k in (6, 40):
    pk = cil.make_params(metric, k, 1.0)
    ws = cil.alloc_workspace(w.m, pk)
    tr[:] = 0
    cil.lib().cil_debug_engine_trace(tr.data_ptr())
    cil.cil_icp_run(t, src, d(np.eye(4)), pk, ws=ws)
    torch.cuda.synchronize()
    cil.lib().cil_debug_engine_trace(None)
    a = tr.cpu().numpy().reshape(-1, 16)
    for it in ((k - 1,) if k < 10 else (k - 3, k - 2, k - 1)):
        sel = (a[:, 8] != 0) & (a[:, 13] == it)
        r = a[sel]
        if len(r) == 0:
            print("cert run iteration", it, "no searched slots"); continue
        fl = r[:, 0]
        ck = r[:, 8:13].astype(np.float64)
        tot = ck.sum(1)
        print(f"cert run iteration {it}: searched slots {len(r)}, active lanes/packet mean {r[:, 14].mean():.1f}, "
              f"normal {(fl & 1).mean():.3f} outlier {((fl >> 1) & 1).mean():.3f} overflow {((fl >> 2) & 1).mean():.3f} "
              f"sparse {((fl >> 3) & 1).mean():.3f}")
        print(f"   clocks per packet (lane view) p50 {np.percentile(tot, 50):.0f} p90 {np.percentile(tot, 90):.0f} max {tot.max():.0f}; "
              f"mean share A,B,C,DE,F {(ck.sum(0) / ck.sum()).round(3).tolist()}; nF mean {r[:, 4].mean():.1f} items mean {r[:, 6].mean():.1f}")
