"""Debug the certified warm start on reduced C4: first iteration where cil_icp_run with
certificates differs from the run without; dump the differing queries' certificate state."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1807_00399_b200 as cil
from tests import workloads as W

def al(x): return (x + 255) // 256 * 256
def layout(m):
    L = {}
    L["partials"] = 256
    L["apose"] = L["partials"] + al(1184 * 32 * 8)
    L["adelta"] = L["apose"] + al(256 * 12 * 8)
    L["nn"] = L["adelta"] + al(256 * 16 * 4)
    L["gw"] = L["nn"] + al(m * 4)
    L["pmask"] = L["gw"] + al(m * 4)
    L["plist"] = L["pmask"] + al((m + 31) // 32 * 4)
    L["gs"] = L["plist"] + al((m + 31) // 32 * 4)
    L["gd1"] = L["gs"] + al(m * 4)
    L["gp"] = L["gd1"] + al(m * 4)
    L["vlist"] = L["gp"] + al(m * 4)
    return L

metric = "point_to_plane"
w = W.c4(metric, rings=16, az=8000)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src = d(w.source)
L = layout(w.m)
def run(k, cert):
    cil.set_certificates(cert)
    prm = cil.make_params(metric, k, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm)
    res, _ = cil.cil_icp_run(t, src, d(np.eye(4)), prm, ws=ws)
    torch.cuda.synchronize()
    return cil.decode_result(res), ws
for k in range(1, 21):
    a, wa = run(k, True)
    b, wb = run(k, False)
    if not np.array_equal(a.pose, b.pose):
        print("first differing run length", k, flush=True)
        break
else:
    print("no difference in 20 iterations"); sys.exit()
nn_a = wa[L["nn"]:L["nn"] + 4 * w.m].view(torch.int32).cpu().numpy()
nn_b = wb[L["nn"]:L["nn"] + 4 * w.m].view(torch.int32).cpu().numpy()
prev, _ = run(k - 1, False)
P = prev.pose
s = (w.source.astype(np.float64) @ P[:3, :3].T) + P[:3, 3]
diff = np.nonzero(nn_a != nn_b)[0]
print("differing queries", len(diff), flush=True)
# the certificate state that k-1 iterations with certificates left behind
_, wc = run(k - 1, True)
gw = wc[L["gw"]:L["gw"] + 4 * w.m].view(torch.int32).cpu().numpy().view(np.uint32)
gs = wc[L["gs"]:L["gs"] + 4 * w.m].view(torch.float32).cpu().numpy()
vl = wc[L["vlist"]:L["vlist"] + 32 * w.m].view(torch.int32).cpu().numpy().reshape(w.m, 8)
nnc = wc[L["nn"]:L["nn"] + 4 * w.m].view(torch.int32).cpu().numpy()
T64 = w.target.astype(np.float64)
info = t.info()
for q in diff[:8]:
    dd = ((T64 - s[q]) ** 2).sum(1)
    o = np.argsort(dd)[:3]
    G1 = (gw[q] & ~np.uint32(255)).view(np.float32)
    print(f"q {q}: cert nn {nn_a[q]} full nn {nn_b[q]} brute {o[0]} d2 {dd[o[0]]:.6g},{dd[o[1]]:.6g} | prev nn {nnc[q]} "
          f"slot {gw[q] & 255} G1 {G1:.4g} GS {gs[q]:.4g} list {vl[q].tolist()}", flush=True)
