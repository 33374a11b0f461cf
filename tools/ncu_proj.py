"""One C3 projective run (30 iterations, point-to-plane) for ncu captures of icp_proj_kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w = gen.c3_depth()
K = cil.make_intrinsics(gen.W, gen.H, gen.FX, gen.FY, gen.CX, gen.CY)
tg = d(w.target)
t3 = cil.cil_target_build(tg, None)
n3, _ = cil.cil_estimate_normals(t3, 10, (0.0, 0.0, 0.0))
prm = cil.make_params("point_to_plane", 30, w.max_dist)
res, _ = cil.cil_proj_run(tg, n3, K, d(w.source), d(np.eye(4)), prm)
torch.cuda.synchronize()
print("ok", cil.decode_result(res).n_corr)
