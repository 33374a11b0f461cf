import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil
d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w5 = gen.c5_patches(int(sys.argv[1]))
t5 = cil.cil_target_build(d(w5.target), d(w5.target_normals)); s5 = d(w5.source)
p5 = cil.make_params("point_to_plane", 1, w5.max_dist); ws5 = cil.alloc_workspace(w5.m, p5)
for _ in range(2):
    cil.cil_icp_iterate(t5, s5, d(np.eye(4)), p5, ws=ws5, want_sys=False)
torch.cuda.synchronize()
print("ok")
