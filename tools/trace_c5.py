"""Engine trace on C5 (one iteration at the identity pose)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
logn = int(sys.argv[1]) if len(sys.argv) > 1 else 20
w = gen.c5_patches(logn)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src = d(w.source)
prm = cil.make_params("point_to_plane", 1, w.max_dist)
tr = torch.zeros(w.m * 16, dtype=torch.int32, device="cuda")
cil.lib().cil_debug_engine_trace(tr.data_ptr())
cil.cil_icp_iterate(t, src, d(np.eye(4)), prm, want_sys=False)
torch.cuda.synchronize()
cil.lib().cil_debug_engine_trace(None)
a = tr.cpu().numpy().reshape(-1, 16)
f32 = lambda x: np.asarray(x, np.int32).view(np.float32)
fl = a[:, 0]; lane0 = np.arange(len(a)) % 32 == 0
q = lambda x: np.percentile(x, [50, 90, 99]).round(3).tolist()
print(f"C5 2^{logn}: normal {(fl & 1).mean():.3f} outlier {((fl >> 1) & 1).mean():.3f} overflow {((fl >> 2) & 1).mean():.3f} sparse {((fl >> 3) & 1).mean():.3f}")
print("  r after hint p50/90/99", q(f32(a[:, 1])), " final d p50/90/99", q(np.sqrt(f32(a[:, 7]))))
print("  nF per packet p50/90/99", q(a[lane0, 4]), " items/query p50/90/99", q(a[:, 6]))
ck = a[lane0, 8:13].astype(np.float64)
print("  clock share A,B,C,DE,F", (ck.sum(0) / ck.sum()).round(3).tolist(), "mean clocks/packet", round(ck.sum() / lane0.sum()))
