"""Small driver for ncu captures: build the C4 target and run cil_icp_run once."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
metric = sys.argv[1] if len(sys.argv) > 1 else "point_to_plane"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
leaf = int(sys.argv[3]) if len(sys.argv) > 3 else 8
w = gen.c4_lidar(metric)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
t = cil.cil_target_build(d(w.target), d(w.target_normals), leaf)
prm = cil.make_params(metric, iters, 1.0)
res, _ = cil.cil_icp_run(t, d(w.source), d(np.eye(4)), prm)
r = cil.decode_result(res)
print("status", r.status, "n_corr", r.n_corr, "rmse", r.rmse)
