"""ncu target: one C4 cil_icp_run of N iterations with certificates (steady-state kernels)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 42
w = gen.c4_lidar("point_to_plane")
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals))
prm = cil.make_params("point_to_plane", iters, 1.0)
res, _ = cil.cil_icp_run(t, d(w.source), d(np.eye(4)), prm)
torch.cuda.synchronize()
print("ok", cil.decode_result(res).rmse)
