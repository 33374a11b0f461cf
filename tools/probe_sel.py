"""Per-iteration K_sel classification on C4 (diagnostic counters in the workspace state):
point-certified, leaf-evaluated, list-evaluated (+ extra list leaves), searched."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1807_00399_b200 as cil

d = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
w = gen.c4_lidar("point_to_plane")
t = cil.cil_target_build(d(w.target), d(w.target_normals))
src = d(w.source)
prev = np.zeros(5)
ws = None
for k in range(1, 51):
    prm = cil.make_params("point_to_plane", k, w.max_dist)
    ws = cil.alloc_workspace(w.m, prm) if ws is None else ws
    cil.cil_icp_run(t, src, d(np.eye(4)), prm, ws=ws, want_log=False)
    torch.cuda.synchronize()
    st = ws[176:216].cpu().view(torch.int64).numpy().astype(np.float64)   # searched, pcert, leaf, list, items
    cur = st
    dlt = cur - prev
    prev = cur
    m = w.m
    print(f"it {k-1:2d}: searched {dlt[0]/m:6.3f} pointcert {dlt[1]/m:6.3f} leaf {dlt[2]/m:6.3f} list {dlt[3]/m:6.3f} "
          f"extra-list-leaves/pt {dlt[4]/m:6.3f}")
