"""ncu target: a few stateless C4 iterations at a given pose fraction (launch 0 = warm-up)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
from scipy.spatial.transform import Rotation
frac = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
w = gen.c4_lidar("point_to_plane")
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals))
rv = Rotation.from_matrix(w.gt_pose[:3, :3]).as_rotvec() * frac
T = np.eye(4); T[:3, :3] = Rotation.from_rotvec(rv).as_matrix(); T[:3, 3] = w.gt_pose[:3, 3] * frac
prm = cil.make_params("point_to_plane", 1, 1.0)
src, P = d(w.source), d(T)
for _ in range(3):
    cil.cil_icp_iterate(t, src, P, prm, want_sys=False)
torch.cuda.synchronize()
print("ok")
